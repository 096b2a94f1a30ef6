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
  switch (ab) {
    case AFG_F32: e = launch_c<float>(c, a, batch, stream); break;
    case AFG_F16: e = launch_c<__half>(c, a, batch, stream); break;
    default: e = launch_c<__nv_bfloat16>(c, a, batch, stream); break;
  }
  return cuda_status(e, "gemm_simt launch");
}

}  // namespace afg
