// gemm_simt.cu - K1b: fp32 (and any-shape) GEMM on the CUDA cores.
//
// Used for (i) the fp32 config (BASELINE configs[0]: 1024^3 + bias + ReLU,
// the reference CPU path's own operator test) and (ii) shapes the TMA path
// cannot address (row pitch not a multiple of 16 bytes, e.g. the 4x4 / 3x5
// graphs of test_frontend.cpp) and strided batch_matmul.
//
// Numerics: every output element is accumulated by ONE thread, k = 0..K-1 in
// order, with fmaf. The reference interpreter computes
//   C = round_f32(double(a) * double(b) + double(C))        (interp.cpp:335-347)
// per k; the double product of two f32 values is exact, so that is exactly a
// single-rounding fused multiply-add: this kernel reproduces af::interpret
// bit-for-bit on f32 inputs (and the bias add / max epilogue nests are each a
// single f32 rounding too, frontend.cpp:447-459).
#include <cuda_runtime.h>

#include <cstdlib>

#include "afg_internal.h"
#include "epilogue.cuh"

namespace afg {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  return OutCvt<T>::from(*p);
}
template <>
__device__ __forceinline__ float ldf<float>(const float* p) {
  return *p;
}

struct SimtArgs {
  const void* A;
  const void* B;
  const float* bias;
  const void* residual;
  void* C;
  int64_t lda, ldb, ldc;
  int64_t sA, sB, sC;  // batch strides (elements)
  int M, N, K;
  int b_nk;  // B stored [N,K]
  int epi;
};

template <typename TA, typename TC>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtArgs a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int64_t bz = blockIdx.z;
  const TA* A = reinterpret_cast<const TA*>(a.A) + bz * a.sA;
  const TA* B = reinterpret_cast<const TA*>(a.B) + bz * a.sB;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  // Loader mapping: 1024 elements per tile, 4 per thread.
  float ra[4], rb[4];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      // A tile: 64 rows x 16 k, k fastest
      const int am = idx / BK, ak = idx % BK;
      const int gm = m0 + am, gk = k0 + ak;
      ra[e] = (gm < a.M && gk < a.K) ? ldf(A + gm * a.lda + gk) : 0.0f;
      // B tile: 16 k x 64 n
      if (!a.b_nk) {
        const int bk = idx / BN, bn = idx % BN;
        const int gk2 = k0 + bk, gn = n0 + bn;
        rb[e] = (gk2 < a.K && gn < a.N) ? ldf(B + gk2 * a.ldb + gn) : 0.0f;
      } else {
        const int bn = idx / BK, bk = idx % BK;
        const int gk2 = k0 + bk, gn = n0 + bn;
        rb[e] = (gk2 < a.K && gn < a.N) ? ldf(B + gn * a.ldb + gk2) : 0.0f;
      }
    }
  };
  auto store_tiles = [&]() {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      As[idx % BK][idx / BK] = ra[e];
      if (!a.b_nk)
        Bs[idx / BN][idx % BN] = rb[e];
      else
        Bs[idx % BK][idx / BK] = rb[e];
    }
  };

  load_tiles(0);
  for (int k0 = 0; k0 < a.K; k0 += BK) {
    __syncthreads();
    store_tiles();
    __syncthreads();
    if (k0 + BK < a.K) load_tiles(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }

  TC* C = reinterpret_cast<TC*>(a.C) + bz * a.sC;
  const TC* R = a.residual ? reinterpret_cast<const TC*>(a.residual) + bz * a.sC : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= a.N) continue;
      float v = acc[i][j];
      if (a.epi != AFG_EPI_NONE) {
        v = v + a.bias[gn];
        v = apply_act_rt(a.epi, v);
      }
      if (R) v = v + OutCvt<TC>::from(R[gm * a.ldc + gn]);
      C[gm * a.ldc + gn] = OutCvt<TC>::to(v);
    }
  }
}

// fp32 fast path (BASELINE configs[0], the interpreter-exact GEMM): 64 x 64
// tile, 64 threads, an 8 x 8 register block per thread (rows {4ty..4ty+3,
// 32+4ty..}, columns {4tx..4tx+3, 32+4tx..}: every shared-memory read is a
// conflict-free or broadcast LDS.128), 16-deep K slabs double-buffered in
// shared memory with the next slab prefetched into registers. Each output
// still accumulates k = 0..K-1 in order with one fmaf per k -- the
// interpreter's round_f32(a*b + c) per store (interp.cpp:335-347) -- so the
// result stays bit-exact; only the data movement changed (64 FMAs per 4
// LDS.128 instead of 16 per 8 LDS.32).
constexpr int FT = 64, FK = 16;

// TX thread columns x TY thread rows: (8, 8) -> 64 threads, 8x8 outputs each;
// (16, 8) -> 128 threads, 8x4 each; (16, 16) -> 256 threads, 4x4 each (more
// warps to hide the LDS latency, more LDS per FMA).
template <int TX, int TY = 8>
__global__ void __launch_bounds__(TY * TX) gemm_f32_blk_kernel(const SimtArgs a) {
  constexpr int T = TY * TX;           // threads
  constexpr int CN = 64 / TX;          // columns per thread (8 or 4)
  constexpr int RM = 64 / TY;          // rows per thread (8 or 4)
  constexpr int AK = FK * FT / T;      // A values each thread loads per slab
  constexpr int BV = FK * FT / T;      // B values each thread loads per slab
  __shared__ __align__(16) float As[2][FK][FT + 4];
  __shared__ __align__(16) float Bs[2][FK][FT + 4];
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int m0 = blockIdx.y * FT, n0 = blockIdx.x * FT;
  const int64_t bz = blockIdx.z;
  const float* A = reinterpret_cast<const float*>(a.A) + bz * a.sA;
  const float* B = reinterpret_cast<const float*>(a.B) + bz * a.sB;
  float acc[RM][CN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < CN; ++j) acc[i][j] = 0.0f;

  // A: thread reads AK consecutive k of row am; B: BV consecutive columns of row bk
  const int am = tid / (FK / AK), ak0 = (tid % (FK / AK)) * AK;
  const int bk = tid / (FT / BV), bn = (tid % (FT / BV)) * BV;
  float ra[AK], rb[BV];
  auto load = [&](int k0) {
    const int gm = m0 + am;
#pragma unroll
    for (int q = 0; q < AK / 4; ++q) {
      const int gk = k0 + ak0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gm < a.M) {
        if (gk + 3 < a.K) {
          v = *reinterpret_cast<const float4*>(A + static_cast<int64_t>(gm) * a.lda + gk);
        } else {
          const float* p = A + static_cast<int64_t>(gm) * a.lda;
          v.x = gk < a.K ? p[gk] : 0.f;
          v.y = gk + 1 < a.K ? p[gk + 1] : 0.f;
          v.z = gk + 2 < a.K ? p[gk + 2] : 0.f;
        }
      }
      ra[4 * q] = v.x;
      ra[4 * q + 1] = v.y;
      ra[4 * q + 2] = v.z;
      ra[4 * q + 3] = v.w;
    }
    const int gk = k0 + bk;
#pragma unroll
    for (int q = 0; q < BV / 4; ++q) {
      const int gn = n0 + bn + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < a.K && gn < a.N)  // N % 4 == 0 on this path
        v = *reinterpret_cast<const float4*>(B + static_cast<int64_t>(gk) * a.ldb + gn);
      rb[4 * q] = v.x;
      rb[4 * q + 1] = v.y;
      rb[4 * q + 2] = v.z;
      rb[4 * q + 3] = v.w;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int k = 0; k < AK; ++k) As[buf][ak0 + k][am] = ra[k];
#pragma unroll
    for (int q = 0; q < BV / 4; ++q)
      *reinterpret_cast<float4*>(&Bs[buf][bk][bn + 4 * q]) =
          make_float4(rb[4 * q], rb[4 * q + 1], rb[4 * q + 2], rb[4 * q + 3]);
  };
  auto frag = [&](int buf, int kk, float4& a0, float4& a1, float4& b0, float4& b1) {
    a0 = *reinterpret_cast<const float4*>(&As[buf][kk][4 * ty]);
    if constexpr (RM == 8) a1 = *reinterpret_cast<const float4*>(&As[buf][kk][32 + 4 * ty]);
    b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][4 * tx]);
    if constexpr (CN == 8) b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][32 + 4 * tx]);
  };

  load(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < a.K; k0 += FK) {
    const bool more = k0 + FK < a.K;
    if (more) load(k0 + FK);
    // fragments of step kk+1 are read while step kk's FMAs issue
    float4 a0, a1 = make_float4(0.f, 0.f, 0.f, 0.f), b0, b1 = make_float4(0.f, 0.f, 0.f, 0.f);
    frag(buf, 0, a0, a1, b0, b1);
#pragma unroll
    for (int kk = 0; kk < FK; ++kk) {
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      if (kk + 1 < FK) frag(buf, kk + 1, a0, a1, b0, b1);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < CN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  float* C = reinterpret_cast<float*>(a.C) + bz * a.sC;
  const float* R = a.residual ? reinterpret_cast<const float*>(a.residual) + bz * a.sC : nullptr;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int gm = m0 + (i < 4 ? 4 * ty + i : 32 + 4 * ty + i - 4);
    if (gm >= a.M) continue;
#pragma unroll
    for (int h = 0; h < CN / 4; ++h) {
      const int gn = n0 + h * 32 + 4 * tx;
      if (gn >= a.N) continue;
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x = acc[i][4 * h + j];
        if (a.epi != AFG_EPI_NONE) x = apply_act_rt(a.epi, x + a.bias[gn + j]);
        if (R) x = x + R[static_cast<int64_t>(gm) * a.ldc + gn + j];
        v[j] = x;
      }
      *reinterpret_cast<float4*>(C + static_cast<int64_t>(gm) * a.ldc + gn) =
          make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

template <typename TA>
cudaError_t launch_c(afg_dtype c, const SimtArgs& a, int64_t batch, cudaStream_t s) {
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, static_cast<unsigned>(batch));
  switch (c) {
    case AFG_F32: gemm_simt_kernel<TA, float><<<grid, 256, 0, s>>>(a); break;
    case AFG_F16: gemm_simt_kernel<TA, __half><<<grid, 256, 0, s>>>(a); break;
    case AFG_BF16: gemm_simt_kernel<TA, __nv_bfloat16><<<grid, 256, 0, s>>>(a); break;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace

afg_status gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                     const void* residual, void* C, int64_t ldc, int64_t M, int64_t N,
                     int64_t K, int64_t batch, int64_t sA, int64_t sB, int64_t sC,
                     afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                     cudaStream_t stream) {
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31) || batch > 65535)
    return set_error(AFG_ERR_UNSUPPORTED, "gemm_simt: extent too large");
  SimtArgs a;
  a.A = A;
  a.B = B;
  a.bias = bias;
  a.residual = residual;
  a.C = C;
  a.lda = lda;
  a.ldb = ldb;
  a.ldc = ldc;
  a.sA = sA;
  a.sB = sB;
  a.sC = sC;
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(N);
  a.K = static_cast<int>(K);
  a.b_nk = b_layout == AFG_B_NK;
  a.epi = static_cast<int>(epi);
  cudaError_t e;
  // the fp32 8x8-register-block kernel when every row is float4-addressable
  const bool fast = ab == AFG_F32 && c == AFG_F32 && !a.b_nk && lda % 4 == 0 && ldb % 4 == 0 &&
                    ldc % 4 == 0 && N % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(B) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
                    (residual == nullptr || (reinterpret_cast<uintptr_t>(residual) & 15) == 0) &&
                    (sA % 4 == 0) && (sB % 4 == 0) && (sC % 4 == 0);
  static const bool no_fast = [] {  // AFG_SIMT_FAST=0: the general kernel (A/B measurements)
    const char* e = getenv("AFG_SIMT_FAST");
    return e && atoi(e) == 0;
  }();
  if (fast && !no_fast) {
    static const int variant = [] {  // AFG_SIMT_TPB = 64 | 128 (threads per 64x64 tile)
      const char* e = getenv("AFG_SIMT_TPB");
      return e ? atoi(e) : 128;
    }();
    dim3 grid((a.N + FT - 1) / FT, (a.M + FT - 1) / FT, static_cast<unsigned>(batch));
    if (variant == 64)
      gemm_f32_blk_kernel<8><<<grid, 64, 0, stream>>>(a);
    else if (variant == 256)
      gemm_f32_blk_kernel<16, 16><<<grid, 256, 0, stream>>>(a);
    else
      gemm_f32_blk_kernel<16><<<grid, 128, 0, stream>>>(a);
    count_launch();
    return cuda_status(cudaGetLastError(), "gemm_f32_blk launch");
  }
  switch (ab) {
    case AFG_F32: e = launch_c<float>(c, a, batch, stream); break;
    case AFG_F16: e = launch_c<__half>(c, a, batch, stream); break;
    default: e = launch_c<__nv_bfloat16>(c, a, batch, stream); break;
  }
  return cuda_status(e, "gemm_simt launch");
}

}  // namespace afg
