// epilogue.cuh - the fused elementwise tail of the contraction kernels.
//
// Realises the graph chain the reference lowers as separate nests after a
// matmul / conv2d (frontend.cpp:447-500 broadcast_in_dim+add, max(x, zeros)):
//   y = act(acc + bias[n]) (+ residual[m, n])
// applied to the fp32 accumulator before the single store, which is the
// "fusion into copy-out" the paper describes and that the
// reference's own fusion pass never performs (nest 3).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../../include/afg.h"
#include "sm100.cuh"

namespace afg {

__device__ __forceinline__ float gelu_tanh(float x) {
  // x * sigmoid(2u), u = sqrt(2/pi) (x + 0.044715 x^3): the composite the
  // reference graph API expresses with a size-2 softmax.
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  // fast reciprocal division (2 ulp): exp overflow -> 1 + e = inf -> 0, the
  // limit of GELU for large negative x
  return __fdividef(x, 1.0f + __expf(-2.0f * u));
}

// erf by Abramowitz & Stegun 7.1.28, erf(x) = 1 - (1 + a1 x + ... + a6 x^6)^-16
// for x >= 0 (|error| <= 1.6e-6 in fp32, far below the bf16 output ulp and
// within the fp32 epilogue tolerance): one MUFU reciprocal, no exp, no branch.
// libdevice erff (~3x the instructions) made the BERT FFN1 epilogue the bound.
__device__ __forceinline__ float erf_fast(float x) {
  const float ax = fabsf(x);
  float p = fmaf(0.0000430638f, ax, 0.0002765672f);
  p = fmaf(p, ax, 0.0001520143f);
  p = fmaf(p, ax, 0.0092705272f);
  p = fmaf(p, ax, 0.0422820123f);
  p = fmaf(p, ax, 0.0705230784f);
  p = fmaf(p, ax, 1.0f);
  float r = __fdividef(1.0f, p);  // p >= 1; overflow -> r = 0 -> erf = 1
  r *= r;
  r *= r;
  r *= r;
  r *= r;
  return copysignf(1.0f - r, x);
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erf_fast(x * 0.7071067811865476f));
}

template <int EPI>
__device__ __forceinline__ float apply_act(float v) {
  if constexpr (EPI == AFG_EPI_BIAS_RELU) return fmaxf(v, 0.0f);
  if constexpr (EPI == AFG_EPI_BIAS_GELU_TANH) return gelu_tanh(v);
  if constexpr (EPI == AFG_EPI_BIAS_GELU_ERF) return gelu_erf(v);
  return v;
}

// Packed (f32x2) activations for a pair of accumulator values: the same
// formulas as above with the FMA-pipe work in one issue slot per pair -- the
// GEMM epilogue of a short-K GEMM (BERT FFN1, K = 768) is issue-bound.
__device__ __forceinline__ uint64_t gelu_tanh2(uint64_t x) {
  using namespace sm100;
  const uint64_t x2 = fmul2(x, x);
  const uint64_t t = ffma2(x2, f2(0.7978845608028654f * 0.044715f, 0.7978845608028654f * 0.044715f),
                           f2(0.7978845608028654f, 0.7978845608028654f));
  // e = exp(-2u) = 2^(-2 log2(e) u)
  const uint64_t z = fmul2(fmul2(t, x), f2(-2.8853900817779268f, -2.8853900817779268f));
  float z0, z1, x0, x1;
  f2split(z, z0, z1);
  f2split(x, x0, x1);
  float e0, e1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z1));
  return f2(__fdividef(x0, 1.0f + e0), __fdividef(x1, 1.0f + e1));
}

__device__ __forceinline__ uint64_t gelu_erf2(uint64_t x) {
  using namespace sm100;
  float x0, x1;
  f2split(x, x0, x1);
  // |x| / sqrt(2) for both lanes, then A&S 7.1.28 in packed Horner form
  const uint64_t a = fmul2(f2(fabsf(x0), fabsf(x1)), f2(0.7071067811865476f, 0.7071067811865476f));
  uint64_t p = ffma2(f2(0.0000430638f, 0.0000430638f), a, f2(0.0002765672f, 0.0002765672f));
  p = ffma2(p, a, f2(0.0001520143f, 0.0001520143f));
  p = ffma2(p, a, f2(0.0092705272f, 0.0092705272f));
  p = ffma2(p, a, f2(0.0422820123f, 0.0422820123f));
  p = ffma2(p, a, f2(0.0705230784f, 0.0705230784f));
  p = ffma2(p, a, f2(1.0f, 1.0f));
  float p0, p1;
  f2split(p, p0, p1);
  uint64_t r = f2(__fdividef(1.0f, p0), __fdividef(1.0f, p1));
  r = fmul2(r, r);
  r = fmul2(r, r);
  r = fmul2(r, r);
  r = fmul2(r, r);  // (1 + ...)^-16 = 1 - erf(|x| / sqrt 2)
  float r0, r1;
  f2split(r, r0, r1);
  // 0.5 x (1 + erf) with erf carrying the sign of x
  const uint64_t one_p_erf = f2(x0 >= 0.0f ? 2.0f - r0 : r0, x1 >= 0.0f ? 2.0f - r1 : r1);
  return fmul2(fmul2(x, f2(0.5f, 0.5f)), one_p_erf);
}

template <int EPI>
__device__ __forceinline__ uint64_t apply_act2(uint64_t v) {
  if constexpr (EPI == AFG_EPI_BIAS_GELU_TANH) return gelu_tanh2(v);
  if constexpr (EPI == AFG_EPI_BIAS_GELU_ERF) return gelu_erf2(v);
  if constexpr (EPI == AFG_EPI_BIAS_RELU) {
    float a, b;
    sm100::f2split(v, a, b);
    return sm100::f2(fmaxf(a, 0.0f), fmaxf(b, 0.0f));
  }
  return v;
}

// Runtime dispatch over the epilogue kind for kernels that do not template it.
__device__ __forceinline__ float apply_act_rt(int epi, float v) {
  switch (epi) {
    case AFG_EPI_BIAS_RELU: return fmaxf(v, 0.0f);
    case AFG_EPI_BIAS_GELU_TANH: return gelu_tanh(v);
    case AFG_EPI_BIAS_GELU_ERF: return gelu_erf(v);
    default: return v;
  }
}

template <typename T> struct OutCvt;
template <> struct OutCvt<float> {
  static __device__ __forceinline__ float to(float v) { return v; }
  static __device__ __forceinline__ float from(float v) { return v; }
};
template <> struct OutCvt<__nv_bfloat16> {
  static __device__ __forceinline__ __nv_bfloat16 to(float v) { return __float2bfloat16_rn(v); }
  static __device__ __forceinline__ float from(__nv_bfloat16 v) { return __bfloat162float(v); }
};
template <> struct OutCvt<__half> {
  static __device__ __forceinline__ __half to(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ float from(__half v) { return __half2float(v); }
};

}  // namespace afg
