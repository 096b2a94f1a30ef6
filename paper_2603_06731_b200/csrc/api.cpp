// api.cpp - the extern "C" boundary (include/afg.h): argument validation,
// status codes + thread-local error text, device checks, TMA descriptor
// encoding through the driver entry point, launch accounting.
//
// Error behaviour mirrors the reference's exceptions (GraphError /
// InterpError, frontend.h:26-28, interp.h:29-31) as status codes; the C++
// graph executor (graph.cpp) turns them back into exceptions.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "afg_internal.h"

namespace afg {

namespace {
thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
}  // namespace

afg_status set_error(afg_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

afg_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return AFG_OK;
  return set_error(AFG_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e),
                   cudaGetErrorString(e));
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  static thread_local int cached_dev = -1, cached_n = 0;
  if (dev == cached_dev) return cached_n;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cached_dev = dev;
  cached_n = n > 0 ? n : 1;
  return cached_n;
}

int stream_slot(void* stream, int kind, int nslots) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, void*>, int> slots;
  static std::map<std::pair<int, int>, int> used;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, kind, stream);
  auto it = slots.find(key);
  if (it != slots.end()) return it->second;
  int& n = used[{dev, kind}];
  if (n >= nslots) return -1;
  return slots[key] = n++;
}

void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("AFG_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

afg_status make_tmap(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int rank,
                     const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                     CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(AFG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver)");
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t bdim[5], estr[5];
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bdim[i] = box[i];
    estr[i] = 1;
    if (i > 0) gstr[i - 1] = strides_bytes[i - 1];
  }
  CUresult r = fn(map, dt, static_cast<cuuint32_t>(rank), const_cast<void*>(base), gdim, gstr,
                  bdim, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(AFG_ERR_INVALID_ARG,
                     "cuTensorMapEncodeTiled failed (%d): rank %d dims[0]=%llu dims[1]=%llu "
                     "box[0]=%u box[1]=%u base=%p",
                     static_cast<int>(r), rank, static_cast<unsigned long long>(dims[0]),
                     static_cast<unsigned long long>(rank > 1 ? dims[1] : 0), box[0],
                     rank > 1 ? box[1] : 0, base);
  return AFG_OK;
}

afg_status make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                        int elem_bytes, int64_t cols, int64_t rows, int64_t ld, int box_cols,
                        int box_rows, CUtensorMapSwizzle swz) {
  const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
  const uint64_t strides[1] = {static_cast<uint64_t>(ld) * elem_bytes};
  const uint32_t box[2] = {static_cast<uint32_t>(box_cols), static_cast<uint32_t>(box_rows)};
  return make_tmap(map, base, dt, 2, dims, strides, box, swz);
}

afg_status make_tmap_im2col_4d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                               int64_t C, int64_t W, int64_t H, int64_t N, const int* lower,
                               const int* upper, int sw, int sh, int channels, int pixels,
                               int elem_bytes) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn) return set_error(AFG_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable (driver)");
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W),
                              static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(N)};
  const cuuint64_t es = static_cast<cuuint64_t>(elem_bytes);
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * es,
                                 static_cast<cuuint64_t>(C * W) * es,
                                 static_cast<cuuint64_t>(C * W * H) * es};
  const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(sw), static_cast<cuuint32_t>(sh), 1};
  CUresult r = fn(map, dt, 4, const_cast<void*>(base), dims, strides, lower, upper,
                  static_cast<cuuint32_t>(channels), static_cast<cuuint32_t>(pixels), estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(AFG_ERR_INVALID_ARG, "cuTensorMapEncodeIm2col failed (%d)", (int)r);
  // Drivers up to 13.1 mis-encode a flag for tensors under 128 KiB (the same
  // workaround CUTLASS applies, copy_traits_sm90_im2col.hpp).
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && C * W * H * N * static_cast<int64_t>(es) < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return AFG_OK;
}

afg_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "no CUDA device");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10)
    return set_error(AFG_ERR_CUDA, "device %d has compute capability %d.x; afg needs sm_100a",
                     dev, major);
  return AFG_OK;
}

}  // namespace afg

using namespace afg;

extern "C" {

const char* afg_last_error(void) { return g_err; }

const char* afg_version(void) { return "afg 0.1 (sm_100a)"; }

int afg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int count = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major == 10) ++count;
  }
  return count;
}

uint64_t afg_launch_count(void) { return g_launches.load(); }

afg_status afg_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                    const void* residual, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                    afg_dtype ab_dtype, afg_dtype c_dtype, afg_layout b_layout,
                    afg_epilogue epi, void* stream) {
  if (!A || !B || !C) return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: null operand");
  if (M <= 0 || N <= 0 || K <= 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: non-positive extent M=%lld N=%lld K=%lld",
                     (long long)M, (long long)N, (long long)K);
  if (!valid_dtype(ab_dtype) || !valid_dtype(c_dtype))
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: bad dtype");
  if (epi < AFG_EPI_NONE || epi > AFG_EPI_BIAS_GELU_ERF)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: bad epilogue %d", (int)epi);
  if (epi != AFG_EPI_NONE && !bias)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: epilogue needs a bias");
  const int64_t min_lda = K;
  const int64_t min_ldb = b_layout == AFG_B_KN ? N : K;
  if (lda < min_lda || ldb < min_ldb || ldc < N)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm: leading dimension too small");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool tc_ok = (ab_dtype == AFG_BF16 || ab_dtype == AFG_F16) && (lda % 8 == 0) &&
                     (ldb % 8 == 0) && aligned16(A) && aligned16(B) &&
                     (c_dtype == AFG_F32 || c_dtype == ab_dtype) && M < (1ll << 31) &&
                     N < (1ll << 31) && K < (1ll << 31) &&
                     (bias == nullptr || aligned16(bias)) && aligned16(C) &&
                     (residual == nullptr || aligned16(residual)) && ldc % 8 == 0;
  if (tc_ok)
    return gemm_tc(A, lda, B, ldb, bias, residual, C, ldc, M, N, K, ab_dtype, c_dtype, b_layout,
                   epi, s);
  return gemm_simt(A, lda, B, ldb, bias, residual, C, ldc, M, N, K, 1, 0, 0, 0, ab_dtype,
                   c_dtype, b_layout, epi, s);
}

afg_status afg_gemm_batched(const void* A, const void* B, void* C, int64_t batch, int64_t M,
                            int64_t N, int64_t K, afg_dtype ab_dtype, afg_dtype c_dtype,
                            void* stream) {
  if (!A || !B || !C) return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_batched: null operand");
  if (batch <= 0 || M <= 0 || N <= 0 || K <= 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_batched: non-positive extent");
  if (!valid_dtype(ab_dtype) || !valid_dtype(c_dtype))
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_batched: bad dtype");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (batch == 1)
    return afg_gemm(A, K, B, N, nullptr, nullptr, C, N, M, N, K, ab_dtype, c_dtype, AFG_B_KN,
                    AFG_EPI_NONE, stream);
  // 16-bit operands with 16-byte aligned rows and batches: one tcgen05 GEMM
  // per batch entry (each is a persistent launch over its own tiles); large
  // enough entries only, small ones stay one batched SIMT launch
  const int64_t ea = dtype_bytes(ab_dtype), ec = dtype_bytes(c_dtype);
  const bool tc = (ab_dtype == AFG_BF16 || ab_dtype == AFG_F16) &&
                  (c_dtype == AFG_F32 || c_dtype == ab_dtype) && K % 8 == 0 && N % 8 == 0 &&
                  aligned16(A) && aligned16(B) && aligned16(C) && (M * K * ea) % 16 == 0 &&
                  (K * N * ea) % 16 == 0 && (M * N * ec) % 16 == 0 && M * N >= 128 * 256 &&
                  batch <= 64;
  if (tc) {
    for (int64_t b = 0; b < batch; ++b) {
      afg_status st2 = gemm_tc(static_cast<const char*>(A) + b * M * K * ea, K,
                               static_cast<const char*>(B) + b * K * N * ea, N, nullptr, nullptr,
                               static_cast<char*>(C) + b * M * N * ec, N, M, N, K, ab_dtype,
                               c_dtype, AFG_B_KN, AFG_EPI_NONE, s);
      if (st2 != AFG_OK) return st2;
    }
    return AFG_OK;
  }
  return gemm_simt(A, K, B, N, nullptr, nullptr, C, N, M, N, K, batch, M * K, K * N, M * N,
                   ab_dtype, c_dtype, AFG_B_KN, AFG_EPI_NONE, s);
}

}  // extern "C"
