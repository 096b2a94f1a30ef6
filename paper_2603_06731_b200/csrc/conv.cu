// conv.cu - K2: convolution entry points.
//
//  afg_conv2d_nhwc : implicit GEMM (M = B*OH*OW, N = OC, K = KH*KW*C,
//                    SPEC.md:395) on the tcgen05 pipeline of gemm_tc.cu with
//                    an im2col-TMA A loader when C % 64 == 0 and the dtype is
//                    bf16/fp16; 1x1 stride-1 unpadded convs are plain GEMMs
//                    on the NHWC activations. Other shapes run a direct SIMT
//                    kernel with the same NHWC/OHWI contract.
//  afg_conv2d_nchw : the reference's own conv2d op semantics (NCHW / OIHW,
//                    IOHW when transposed; frontend.cpp:752-970 and
//                    convReference, oracles.cpp:78-120), direct, fp32
//                    accumulation, any stride / dilation / begin pad.
//  afg_conv_pack_filter : OIHW -> OHWI repack for the implicit GEMM.
#include <cuda_runtime.h>

#include "afg_internal.h"
#include "epilogue.cuh"

namespace afg {
namespace {

template <typename T>
__device__ __forceinline__ float ldx(const T* p) {
  return OutCvt<T>::from(*p);
}

template <typename T, typename TO>
__global__ void conv_nhwc_direct_kernel(const T* __restrict__ x, const T* __restrict__ w,
                                        const float* __restrict__ bias, TO* __restrict__ y,
                                        int B, int H, int W, int C, int OC, int KH, int KW,
                                        int sh, int sw, int pt, int pl, int dh, int dw, int OH,
                                        int OW, int epi) {
  const int64_t total = static_cast<int64_t>(B) * OH * OW * OC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int oc = static_cast<int>(i % OC);
    int64_t r = i / OC;
    const int ox = static_cast<int>(r % OW);
    r /= OW;
    const int oy = static_cast<int>(r % OH);
    const int b = static_cast<int>(r / OH);
    float acc = 0.0f;
    for (int ky = 0; ky < KH; ++ky) {
      const int iy = oy * sh + ky * dh - pt;
      if (iy < 0 || iy >= H) continue;
      for (int kx = 0; kx < KW; ++kx) {
        const int ix = ox * sw + kx * dw - pl;
        if (ix < 0 || ix >= W) continue;
        const T* xp = x + ((static_cast<int64_t>(b) * H + iy) * W + ix) * C;
        const T* wp = w + ((static_cast<int64_t>(oc) * KH + ky) * KW + kx) * C;
        for (int c = 0; c < C; ++c) acc = fmaf(ldx(xp + c), ldx(wp + c), acc);
      }
    }
    if (epi != AFG_EPI_NONE) acc = apply_act_rt(epi, acc + bias[oc]);
    y[i] = OutCvt<TO>::to(acc);
  }
}

template <typename TI, typename TO>
__global__ void conv_nchw_direct_kernel(const TI* __restrict__ x, const TI* __restrict__ w,
                                        TO* __restrict__ y, int B, int C, int H, int W, int OC,
                                        int KH, int KW, int sh, int sw, int dh, int dw, int pt,
                                        int pl, int transposed, int OH, int OW) {
  const int64_t total = static_cast<int64_t>(B) * OC * OH * OW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ox = static_cast<int>(i % OW);
    int64_t r = i / OW;
    const int oy = static_cast<int>(r % OH);
    r /= OH;
    const int oc = static_cast<int>(r % OC);
    const int b = static_cast<int>(r / OC);
    float acc = 0.0f;
    // loop order (ic, ky, kx) as convReference (oracles.cpp:100-112)
    for (int ic = 0; ic < C; ++ic)
      for (int ky = 0; ky < KH; ++ky)
        for (int kx = 0; kx < KW; ++kx) {
          int iy, ix;
          int64_t widx;
          if (!transposed) {
            iy = oy * sh + ky * dh - pt;
            ix = ox * sw + kx * dw - pl;
            widx = ((static_cast<int64_t>(oc) * C + ic) * KH + ky) * KW + kx;
          } else {
            const int ny = oy + pt - ky * dh, nx = ox + pl - kx * dw;
            if (ny % sh != 0 || nx % sw != 0) continue;
            iy = ny / sh;
            ix = nx / sw;
            widx = ((static_cast<int64_t>(ic) * OC + oc) * KH + ky) * KW + kx;
          }
          if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
          acc = fmaf(ldx(x + ((static_cast<int64_t>(b) * C + ic) * H + iy) * W + ix),
                     ldx(w + widx), acc);
        }
    y[i] = OutCvt<TO>::to(acc);
  }
}

template <typename T>
__global__ void pack_filter_kernel(const T* __restrict__ w, T* __restrict__ out, int OC, int C,
                                   int KH, int KW) {
  const int64_t total = static_cast<int64_t>(OC) * C * KH * KW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // out index (oc, ky, kx, c)
    const int c = static_cast<int>(i % C);
    int64_t r = i / C;
    const int kx = static_cast<int>(r % KW);
    r /= KW;
    const int ky = static_cast<int>(r % KH);
    const int oc = static_cast<int>(r / KH);
    out[i] = w[((static_cast<int64_t>(oc) * C + c) * KH + ky) * KW + kx];
  }
}

unsigned grid_1d(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  return static_cast<unsigned>(g < 1 ? 1 : (g > cap ? cap : g));
}

bool fits_int(int64_t v) { return v >= 0 && v < (1ll << 31); }

}  // namespace
}  // namespace afg

using namespace afg;

extern "C" {

afg_status afg_conv2d_nhwc(const void* x, const void* w, const float* bias, void* y, int64_t B,
                           int64_t H, int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                           int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t dh,
                           int64_t dw, int64_t OH, int64_t OW, afg_dtype dt, afg_epilogue epi,
                           void* stream) {
  return afg_conv2d_nhwc_ex(x, w, bias, y, B, H, W, C, OC, KH, KW, sh, sw, pt, pl, dh, dw, OH, OW,
                            dt, dt, epi, stream);
}

afg_status afg_conv2d_nhwc_ex(const void* x, const void* w, const float* bias, void* y, int64_t B,
                              int64_t H, int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                              int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t dh,
                              int64_t dw, int64_t OH, int64_t OW, afg_dtype dt, afg_dtype yt,
                              afg_epilogue epi, void* stream) {
  if (!x || !w || !y) return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc: null operand");
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || OC <= 0 || KH <= 0 || KW <= 0 || sh <= 0 ||
      sw <= 0 || dh <= 0 || dw <= 0 || OH <= 0 || OW <= 0 || pt < 0 || pl < 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc: bad geometry");
  if ((OH - 1) * sh - pt + (KH - 1) * dh < 0 || (OW - 1) * sw - pl + (KW - 1) * dw < 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc: bad output extent");
  if (!valid_dtype(dt) || !(yt == dt || yt == AFG_F32))
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc: bad dtype pair");
  if (epi != AFG_EPI_NONE && !bias)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nhwc: epilogue needs a bias");
  const int64_t M = B * OH * OW;
  if (!fits_int(M) || !fits_int(B * H * W * C) || !fits_int(KH * KW * C))
    return set_error(AFG_ERR_UNSUPPORTED, "afg_conv2d_nhwc: extent too large");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool tc = (dt == AFG_BF16 || dt == AFG_F16) && C % 64 == 0 && aligned16(x) &&
                  aligned16(w) && (bias == nullptr || aligned16(bias));
  if (tc && KH == 1 && KW == 1 && sh == 1 && sw == 1 && pt == 0 && pl == 0 && OH == H &&
      OW == W) {
    // 1x1 / stride 1: the implicit GEMM is the plain GEMM on [B*H*W, C] x [OC, C]^T
    return gemm_tc(x, C, w, C, bias, nullptr, y, OC, M, OC, C, dt, yt, AFG_B_NK, epi, s);
  }
  if (tc && KH == 3 && KW == 3 && sh == 1 && sw == 1 && dh == 1 && dw == 1 && pt == 1 &&
      pl == 1 && OH == H && OW == W) {
    // 3x3 / stride 1 / pad 1: the input halo is staged once per tile, not per tap
    st = conv_halo(x, w, bias, y, B, H, W, C, OC, dt, yt, epi, s);
    if (st != AFG_ERR_UNSUPPORTED) return st;
  }
  if (tc && sh <= 8 && sw <= 8) {
    st = conv_tc(x, w, bias, y, B, H, W, C, OC, KH, KW, sh, sw, pt, pl, dh, dw, OH, OW, dt, yt, epi,
                 s);
    if (st != AFG_ERR_UNSUPPORTED) return st;
  }
  const unsigned g = grid_1d(M * OC);
#define AFG_DIRECT(T, TO)                                                                      \
  conv_nhwc_direct_kernel<T, TO><<<g, 256, 0, s>>>(                                            \
      reinterpret_cast<const T*>(x), reinterpret_cast<const T*>(w), bias, reinterpret_cast<TO*>(y), \
      (int)B, (int)H, (int)W, (int)C, (int)OC, (int)KH, (int)KW, (int)sh, (int)sw, (int)pt,     \
      (int)pl, (int)dh, (int)dw, (int)OH, (int)OW, (int)epi)
  if (dt == AFG_F32) AFG_DIRECT(float, float);
  else if (dt == AFG_F16 && yt == AFG_F32) AFG_DIRECT(__half, float);
  else if (dt == AFG_F16) AFG_DIRECT(__half, __half);
  else if (yt == AFG_F32) AFG_DIRECT(__nv_bfloat16, float);
  else AFG_DIRECT(__nv_bfloat16, __nv_bfloat16);
#undef AFG_DIRECT
  count_launch();
  return cuda_status(cudaGetLastError(), "conv_nhwc_direct launch");
}

afg_status afg_conv2d_nchw(const void* x, const void* w, void* y, int64_t B, int64_t C,
                           int64_t H, int64_t W, int64_t OC, int64_t KH, int64_t KW, int64_t sh,
                           int64_t sw, int64_t dh, int64_t dw, int64_t pt, int64_t pl,
                           int transposed, int64_t OH, int64_t OW, afg_dtype xd, afg_dtype yd,
                           void* stream) {
  if (!x || !w || !y) return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nchw: null operand");
  if (B <= 0 || C <= 0 || H <= 0 || W <= 0 || OC <= 0 || KH <= 0 || KW <= 0 || sh <= 0 ||
      sw <= 0 || dh <= 0 || dw <= 0 || OH <= 0 || OW <= 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nchw: bad geometry");
  if (!valid_dtype(xd) || !valid_dtype(yd))
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv2d_nchw: bad dtype");
  if (!fits_int(B * C * H * W) || !fits_int(B * OC * OH * OW))
    return set_error(AFG_ERR_UNSUPPORTED, "afg_conv2d_nchw: extent too large");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = grid_1d(B * OC * OH * OW);
#define AFG_NCHW(TI, TO)                                                                     \
  conv_nchw_direct_kernel<TI, TO><<<g, 256, 0, s>>>(                                         \
      reinterpret_cast<const TI*>(x), reinterpret_cast<const TI*>(w), reinterpret_cast<TO*>(y), \
      (int)B, (int)C, (int)H, (int)W, (int)OC, (int)KH, (int)KW, (int)sh, (int)sw, (int)dh,   \
      (int)dw, (int)pt, (int)pl, transposed, (int)OH, (int)OW)
  if (xd == AFG_F32 && yd == AFG_F32) AFG_NCHW(float, float);
  else if (xd == AFG_F16 && yd == AFG_F32) AFG_NCHW(__half, float);
  else if (xd == AFG_F16 && yd == AFG_F16) AFG_NCHW(__half, __half);
  else if (xd == AFG_BF16 && yd == AFG_F32) AFG_NCHW(__nv_bfloat16, float);
  else if (xd == AFG_BF16 && yd == AFG_BF16) AFG_NCHW(__nv_bfloat16, __nv_bfloat16);
  else if (xd == AFG_F32 && yd == AFG_F16) AFG_NCHW(float, __half);
  else return set_error(AFG_ERR_UNSUPPORTED, "afg_conv2d_nchw: dtype pair");
#undef AFG_NCHW
  count_launch();
  return cuda_status(cudaGetLastError(), "conv_nchw_direct launch");
}

afg_status afg_conv_pack_filter(const void* w, void* out, int64_t OC, int64_t C, int64_t KH,
                                int64_t KW, afg_dtype dt, void* stream) {
  if (!w || !out || OC <= 0 || C <= 0 || KH <= 0 || KW <= 0 || !valid_dtype(dt))
    return set_error(AFG_ERR_INVALID_ARG, "afg_conv_pack_filter: bad arguments");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = grid_1d(OC * C * KH * KW);
  if (dt == AFG_F32)
    pack_filter_kernel<float><<<g, 256, 0, s>>>(reinterpret_cast<const float*>(w),
                                                reinterpret_cast<float*>(out), (int)OC, (int)C,
                                                (int)KH, (int)KW);
  else
    pack_filter_kernel<uint16_t><<<g, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(w),
                                                   reinterpret_cast<uint16_t*>(out), (int)OC,
                                                   (int)C, (int)KH, (int)KW);
  count_launch();
  return cuda_status(cudaGetLastError(), "pack_filter launch");
}

}  // extern "C"
