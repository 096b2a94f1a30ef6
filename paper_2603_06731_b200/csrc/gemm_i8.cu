// K1c — int8 GEMM on the 5th-generation tensor cores (tcgen05 kind::i8).
//
// The quant module's repositioned form (PAPER.md Appendix
// A.1): dequant(Qa) . dequant(Qb) -> quant becomes an i8 x i8 matmul with an
// exact i32 accumulator and the combined scale applied once at the output.
// Output modes (afg.h): the i32 accumulator itself (bit-exact vs the integer
// oracle), a requantised i8 (round half away from zero, saturating — the
// interpreter's `quant`, test_interp.cpp:286-307), or the dequantised f32.
//
// Structure (same pipeline as K1, gemm_tc.cu): persistent CTA per SM, warp 0
// streams 128-byte K slabs of A [128 rows] and B [256 rows, K-major] with TMA
// (128B swizzle) into a 4-deep ring, warp 1 issues 128 x 256 x 32 MMAs (one
// elected lane, warp-uniform loop; 256 x 256 x 32 on a CTA pair with a 6-deep
// ring of half-B stages when the tiles fill the GPU), warp 2 owns 512 TMEM columns (two
// 256-column s32 accumulators: the epilogue of tile i overlaps the MMAs of
// tile i+1), warps 4-11 (two warpgroups, alternate 32-column chunks) read the
// accumulator rows back (one row per thread) and store them. Requantised /
// dequantised outputs round exactly like the reference's double arithmetic
// (interp.cpp:502-561): fp32 with an error-free product residual where that is
// provably identical, double otherwise.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "afg_internal.h"
#include "sm100.cuh"

namespace afg {
namespace {

using namespace sm100;

constexpr int I8_BM = 128;
constexpr int I8_BN = 256;
constexpr int I8_BK = 128;  // K elements (= bytes) per stage: one 128-byte swizzle row
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 x 256 tile
// with one M = 256 MMA per K step; each CTA stages its 128 rows of A and half
// of B (as K1's pair tiles): half the B bytes per SM in smem and L2.
template <bool PAIR>
struct I8Smem {
  static constexpr int STAGES = PAIR ? 6 : 4;
  static constexpr int B_ROWS = PAIR ? I8_BN / 2 : I8_BN;
  static constexpr int A_BYTES = I8_BM * I8_BK;
  static constexpr int B_BYTES = B_ROWS * I8_BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 4;
  static constexpr int TOTAL = BAR_OFF + NUM_BARS * 8 + 16 + 1024;
  static_assert(TOTAL <= 232448, "gemm_i8 smem");
};

struct I8Args {
  int M, N, K;
  int64_t ldc;  // elements of the output type
  void* C;
  int mode;  // 0 i32, 1 requantised i8, 2 dequantised f32
  double scale;
  float scale_f;  // the same value (the C ABI passes a float)
  int nmb, nnb;
  // implicit-GEMM conv (IM2COL): K slab kb = (filter tap, 128-channel block)
  int c_blocks, taps, KW, dil_w, dil_h, OH, OW, stride_w, stride_h, lower_w, lower_h;
};

// tcgen05 instruction descriptor, kind::i8: D = s32, A = B = signed 8-bit,
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int CG>
__device__ __forceinline__ void mma_i8_if(bool leader, uint32_t tmem_d, uint64_t adesc,
                                          uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::%6.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(static_cast<uint32_t>(leader)),
      "n"(CG)
      : "memory");
}

// round half away from zero, saturate to [-128, 127] (interp quant), in double
__device__ __forceinline__ int requant_i8(int acc, double scale) {
  const double r = round(static_cast<double>(acc) * scale);
  return static_cast<int>(fmin(fmax(r, -128.0), 127.0));
}

// The same result in fp32, exactly: for |acc| < 2^24 the float acc is exact,
// y = acc * s is the correctly rounded product and e = fma(acc, s, -y) its
// exact residual (acc * s = y + e). Rounding y + e half away from zero only
// needs e at an exact .5 fraction of y (elsewhere |f| <= 0.5 - ulp(y) and
// |e| <= ulp(y) / 2 cannot cross the boundary). Larger |acc|: the double path.
__device__ __forceinline__ int requant_i8_fast(int acc, float s, double sd) {
  if (acc > -(1 << 24) && acc < (1 << 24)) {
    const float a = static_cast<float>(acc);
    const float y = a * s;
    const float e = fmaf(a, s, -y);
    const float r = truncf(y);
    const float f = fabsf(y - r);
    const bool away = f > 0.5f || (f == 0.5f && (e == 0.0f || (e > 0.0f) == (y > 0.0f)));
    const float q = away ? r + copysignf(1.0f, y) : r;
    return static_cast<int>(fminf(fmaxf(q, -128.0f), 127.0f));
  }
  return requant_i8(acc, sd);
}

// (float)(acc * scale) as the reference computes it (double product, one
// rounding to f32): for |acc| < 2^24 the double product is exact, so the fp32
// product (one correct rounding) is the same value.
__device__ __forceinline__ float dequant_f32(int acc, float s, double sd) {
  if (acc > -(1 << 24) && acc < (1 << 24)) return static_cast<float>(acc) * s;
  return static_cast<float>(static_cast<double>(acc) * sd);
}

__device__ __forceinline__ void store_row32(const uint32_t (&r)[32], const I8Args& a, int row,
                                            int col0) {
  if (row >= a.M || col0 >= a.N) return;
  const bool full = col0 + 32 <= a.N;
  if (a.mode == 0) {
    int32_t* dst = static_cast<int32_t*>(a.C) + static_cast<int64_t>(row) * a.ldc + col0;
    if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
      for (int v = 0; v < 8; ++v)
        reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) dst[j] = static_cast<int32_t>(r[j]);
    }
  } else if (a.mode == 1) {
    int8_t* dst = static_cast<int8_t*>(a.C) + static_cast<int64_t>(row) * a.ldc + col0;
    uint32_t w[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      uint32_t x = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        x |= (static_cast<uint32_t>(requant_i8_fast(static_cast<int>(r[4 * v + b]), a.scale_f,
                                                     a.scale)) &
              0xffu)
             << (8 * b);
      w[v] = x;
    }
    if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) dst[j] = static_cast<int8_t>((w[j / 4] >> (8 * (j % 4))) & 0xffu);
    }
  } else {
    float* dst = static_cast<float*>(a.C) + static_cast<int64_t>(row) * a.ldc + col0;
    float f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      f[j] = dequant_f32(static_cast<int>(r[j]), a.scale_f, a.scale);
    if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
      for (int v = 0; v < 8; ++v)
        reinterpret_cast<float4*>(dst)[v] = make_float4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) dst[j] = f[j];
    }
  }
}

template <bool PAIR, bool IM2COL = false>
__global__ void __launch_bounds__(384, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const I8Args args) {
  static_assert(!(PAIR && IM2COL), "the int8 conv runs single-CTA tiles");
  using L = I8Smem<PAIR>;
  constexpr int NS = L::STAGES;
  constexpr int TILE_M = PAIR ? 2 * I8_BM : I8_BM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + NS;
  uint64_t* tfull_bar = bars + 2 * NS;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NUM_BARS);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int cid = PAIR ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int ncl = PAIR ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      // PAIR: one arrival per epilogue warp of both CTAs (on the leader's)
      mbar_init(&tempty_bar[s], PAIR ? 16 : 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  griddep_launch_dependents();

  const int num_tiles = args.nmb * args.nnb;
  const int num_kb = IM2COL ? args.taps * args.c_blocks : (args.K + I8_BK - 1) / I8_BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        const int m0 = (t % args.nmb) * TILE_M + static_cast<int>(rank) * I8_BM;
        const int n0 = (t / args.nmb) * I8_BN + static_cast<int>(rank) * L::B_ROWS;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          // PAIR: both CTAs' bytes complete on the leader's full barrier
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], (PAIR ? 2 : 1) * L::STAGE_BYTES);
          if constexpr (IM2COL) {
            // 128 output pixels x 128 channels of one filter tap, gathered by
            // the TMA unit in im2col mode (zero fill = padding / channel tail);
            // B = the OHWI filter as [OC, taps, C] (channel tail zero-filled)
            const int q = m0 % args.OW;
            const int p = (m0 / args.OW) % args.OH;
            const int n = m0 / (args.OW * args.OH);
            const int tap = kb / args.c_blocks;
            const int cb = kb - tap * args.c_blocks;
            const int ky = tap / args.KW;
            const int kx = tap - ky * args.KW;
            tma_load_im2col_4d(sa, &tmA, &full_bar[stage], cb * I8_BK,
                               args.lower_w + q * args.stride_w, args.lower_h + p * args.stride_h,
                               n, static_cast<uint16_t>(kx * args.dil_w),
                               static_cast<uint16_t>(ky * args.dil_h));
            tma_load_3d(sa + L::A_BYTES, &tmB, &full_bar[stage], cb * I8_BK, tap, n0);
          } else if constexpr (PAIR) {
            const uint32_t fb = mapa_shared(&full_bar[stage], 0);
            tma_load_2d_pair(sa, &tmA, fb, kb * I8_BK, m0);
            tma_load_2d_pair(sa + L::A_BYTES, &tmB, fb, kb * I8_BK, n0);
          } else {
            tma_load_2d(sa, &tmA, &full_bar[stage], kb * I8_BK, m0);
            tma_load_2d(sa + L::A_BYTES, &tmB, &full_bar[stage], kb * I8_BK, n0);
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // PAIR: the leader CTA issues for both
      const bool leader = elect_one();
      constexpr uint32_t idesc = idesc_i8(TILE_M, I8_BN);
      const uint64_t a_desc0 = desc_kmajor_sw128(smem_u32(smem));
      const uint64_t b_desc0 = desc_kmajor_sw128(smem_u32(smem + L::A_BYTES));
      constexpr uint64_t STAGE_STEP = L::STAGE_BYTES >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int t = cid; t < num_tiles; t += ncl, ++iter) {
        const int acc = iter & 1;
        if constexpr (PAIR) mbar_wait_cluster(&tempty_bar[acc], ((iter >> 1) & 1) ^ 1);
        else mbar_wait(&tempty_bar[acc], ((iter >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * I8_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage) * STAGE_STEP;
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage) * STAGE_STEP;
#pragma unroll
          for (int k = 0; k < I8_BK / 32; ++k)  // 32 bytes of K per MMA
            mma_i8_if<PAIR ? 2 : 1>(leader, d_tmem, ad + static_cast<uint64_t>((k * 32) >> 4),
                                    bd + static_cast<uint64_t>((k * 32) >> 4), idesc,
                                    (kb | k) != 0 ? 1u : 0u);
          if constexpr (PAIR) mma_commit_pair_if(leader, &empty_bar[stage], 3);
          else mma_commit_if(leader, &empty_bar[stage]);
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (PAIR) mma_commit_pair_if(leader, &tfull_bar[acc], 3);
        else mma_commit_if(leader, &tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // two epilogue warpgroups (warps 4-7, 8-11) take alternate 32-column chunks
    const int eg = (warp - 4) / 4;
    const int ew = warp % 4;
    const int rloc = ew * 32 + lane;
    int iter = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++iter) {
      const int acc = iter & 1;
      mbar_wait(&tfull_bar[acc], (iter >> 1) & 1);
      tc_fence_after();
      const int row = (t % args.nmb) * TILE_M + static_cast<int>(rank) * I8_BM + rloc;
      const int n0 = (t / args.nmb) * I8_BN;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * I8_BN;
#pragma unroll 1
      for (int c = eg; c < I8_BN / 32; c += 2) {
        uint32_t r[32];
        tmem_ld32(t_row + c * 32, r);
        tmem_wait_ld();
        if (c + 2 >= I8_BN / 32) {  // last TMEM read of the tile: release the accumulator
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
        }
        store_row32(r, args, row, n0 + c * 32);
      }
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // the leader's MMAs into the peer's TMEM are done
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

template <bool PAIR, bool IM2COL = false>
cudaError_t launch_i8(const CUtensorMap& tmA, const CUtensorMap& tmB, const I8Args& a,
                      cudaStream_t stream) {
  constexpr int smem = I8Smem<PAIR>::TOTAL;
  static std::atomic<uint64_t> configured{0};  // per instantiation, one bit per device
  if (cudaError_t e = ensure_smem_optin(configured, gemm_i8_kernel<PAIR, IM2COL>, smem);
      e != cudaSuccess)
    return e;
  const int tiles = a.nmb * a.nnb;
  const int grid = PAIR ? 2 * std::min(tiles, num_sms() / 2) : std::min(tiles, num_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(384);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_i8_kernel<PAIR, IM2COL>, tmA, tmB, a);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

afg_status gemm_i8(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                   int64_t M, int64_t N, int64_t K, int mode, double scale, cudaStream_t stream) {
  // 256 x 256 tiles on CTA pairs when they fill at least half the SMs' pairs
  // (AFG_GEMM_I8_PAIR=0 keeps single-CTA 128 x 256 tiles)
  static const bool pair_env = [] {
    const char* e = getenv("AFG_GEMM_I8_PAIR");
    return !(e && atoi(e) == 0);
  }();
  const bool pair = pair_env && M >= 256 && N >= 256 &&
                    ((M + 255) / 256) * ((N + 255) / 256) >= num_sms() / 2;
  CUtensorMap tmA, tmB;
  afg_status st = make_tmap_2d(&tmA, A, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, M, lda, I8_BK, I8_BM);
  if (st != AFG_OK) return st;
  st = make_tmap_2d(&tmB, B, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, N, ldb, I8_BK,
                    pair ? I8_BN / 2 : I8_BN);
  if (st != AFG_OK) return st;
  I8Args a;
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(N);
  a.K = static_cast<int>(K);
  a.ldc = ldc;
  a.C = C;
  a.mode = mode;
  a.scale = scale;
  a.scale_f = static_cast<float>(scale);
  a.nmb = static_cast<int>((M + (pair ? 2 : 1) * I8_BM - 1) / ((pair ? 2 : 1) * I8_BM));
  a.nnb = static_cast<int>((N + I8_BN - 1) / I8_BN);
  const cudaError_t e = pair ? launch_i8<true>(tmA, tmB, a, stream) : launch_i8<false>(tmA, tmB, a, stream);
  return cuda_status(e, "gemm_i8 launch");
}

// int8 implicit-GEMM convolution (NHWC activations, OHWI filter), the conv
// half of the quant path: M = B*OH*OW output pixels, N = OC, K = taps x C.
afg_status conv_i8(const void* x, const void* w, void* y, int64_t B, int64_t H, int64_t W,
                   int64_t C, int64_t OC, int64_t KH, int64_t KW, int64_t sh, int64_t sw,
                   int64_t pt, int64_t pl, int64_t dh, int64_t dw, int64_t OH, int64_t OW,
                   int mode, double scale, cudaStream_t stream) {
  const int64_t pb = (OH - 1) * sh + (KH - 1) * dh + 1 - H - pt;
  const int64_t pr = (OW - 1) * sw + (KW - 1) * dw + 1 - W - pl;
  const int lower[2] = {static_cast<int>(-pl), static_cast<int>(-pt)};
  const int upper[2] = {static_cast<int>(pr - (KW - 1) * dw), static_cast<int>(pb - (KH - 1) * dh)};
  for (int i = 0; i < 2; ++i)
    if (lower[i] < -128 || lower[i] > 127 || upper[i] < -128 || upper[i] > 127)
      return set_error(AFG_ERR_UNSUPPORTED, "conv_i8: padding outside the im2col corner range");
  if (sh > 8 || sw > 8) return set_error(AFG_ERR_UNSUPPORTED, "conv_i8: stride > 8");
  CUtensorMap tmA, tmB;
  afg_status st = make_tmap_im2col_4d(&tmA, x, CU_TENSOR_MAP_DATA_TYPE_UINT8, C, W, H, B, lower,
                                      upper, static_cast<int>(sw), static_cast<int>(sh), I8_BK,
                                      I8_BM, 1);
  if (st != AFG_OK) return st;
  const uint64_t dims[3] = {static_cast<uint64_t>(C), static_cast<uint64_t>(KH * KW),
                            static_cast<uint64_t>(OC)};
  const uint64_t strides[2] = {static_cast<uint64_t>(C), static_cast<uint64_t>(KH * KW * C)};
  const uint32_t box[3] = {static_cast<uint32_t>(I8_BK), 1u, static_cast<uint32_t>(I8_BN)};
  st = make_tmap(&tmB, w, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dims, strides, box,
                 CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != AFG_OK) return st;
  I8Args a{};
  const int64_t M = B * OH * OW;
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(OC);
  a.K = static_cast<int>(KH * KW * C);
  a.ldc = OC;
  a.C = y;
  a.mode = mode;
  a.scale = scale;
  a.scale_f = static_cast<float>(scale);
  a.nmb = static_cast<int>((M + I8_BM - 1) / I8_BM);
  a.nnb = static_cast<int>((OC + I8_BN - 1) / I8_BN);
  a.c_blocks = static_cast<int>((C + I8_BK - 1) / I8_BK);
  a.taps = static_cast<int>(KH * KW);
  a.KW = static_cast<int>(KW);
  a.dil_w = static_cast<int>(dw);
  a.dil_h = static_cast<int>(dh);
  a.OH = static_cast<int>(OH);
  a.OW = static_cast<int>(OW);
  a.stride_w = static_cast<int>(sw);
  a.stride_h = static_cast<int>(sh);
  a.lower_w = lower[0];
  a.lower_h = lower[1];
  return cuda_status(launch_i8<false, true>(tmA, tmB, a, stream), "conv_i8 launch");
}

}  // namespace afg

using namespace afg;

extern "C" afg_status afg_gemm_i8(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                  int64_t ldc, int64_t M, int64_t N, int64_t K, int out_mode,
                                  float scale, void* stream) {
  if (!A || !B || !C) return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_i8: null operand");
  if (M <= 0 || N <= 0 || K <= 0 || M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 17))
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_i8: extent out of range (K < 131072 keeps i32 exact)");
  if (out_mode < 0 || out_mode > 2)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_i8: bad out_mode %d", out_mode);
  if (out_mode != 0 && !(scale > 0.0f))
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_i8: scale must be positive");
  if (lda < K || ldb < K || ldc < N)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_i8: leading dimension too small");
  if (lda % 16 != 0 || ldb % 16 != 0 || !aligned16(A) || !aligned16(B))
    return set_error(AFG_ERR_UNSUPPORTED,
                     "afg_gemm_i8: A / B need 16-byte aligned bases and row pitches (TMA)");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  return gemm_i8(A, lda, B, ldb, C, ldc, M, N, K, out_mode, static_cast<double>(scale),
                 static_cast<cudaStream_t>(stream));
}

extern "C" afg_status afg_conv2d_nhwc_i8(const void* x, const void* w, void* y, int64_t B, int64_t H,
                                         int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                                         int64_t stride_h, int64_t stride_w, int64_t pad_top,
                                         int64_t pad_left, int64_t dil_h, int64_t dil_w, int64_t OH,
                                         int64_t OW, int out_mode, float scale, void* stream) {
  if (!x || !w || !y) return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc_i8: null operand");
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || OC <= 0 || KH <= 0 || KW <= 0 || OH <= 0 ||
      OW <= 0 || stride_h <= 0 || stride_w <= 0 || dil_h <= 0 || dil_w <= 0 || pad_top < 0 ||
      pad_left < 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc_i8: bad geometry");
  if (out_mode < 0 || out_mode > 2)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc_i8: bad out_mode %d", out_mode);
  if (out_mode != 0 && !(scale > 0.0f))
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc_i8: scale must be positive");
  if (KH * KW * C >= (1ll << 17) || B * OH * OW >= (1ll << 31))
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc_i8: extent out of range");
  if (C % 16 != 0 || !aligned16(x) || !aligned16(w))
    return set_error(AFG_ERR_UNSUPPORTED,
                     "afg_conv2d_nhwc_i8: C must be a multiple of 16 with 16-byte aligned bases");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  return conv_i8(x, w, y, B, H, W, C, OC, KH, KW, stride_h, stride_w, pad_top, pad_left, dil_h,
                 dil_w, OH, OW, out_mode, static_cast<double>(scale),
                 static_cast<cudaStream_t>(stream));
}
