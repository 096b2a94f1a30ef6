// afg_internal.h - host-side plumbing shared by the kernels' launchers and the
// C ABI (api.cpp): status/error reporting, device properties, TMA descriptor
// encoding, launch accounting, and the internal per-family entry points.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/afg.h"

namespace afg {

// Sets the thread-local error message and returns `st`.
afg_status set_error(afg_status st, const char* fmt, ...);
// AFG_OK for cudaSuccess, else AFG_ERR_CUDA with the CUDA error text.
afg_status cuda_status(cudaError_t e, const char* what);

int num_sms();              // SM count of the current device
// A counter slot in [0, nslots) owned by (current device, stream) for the
// kernels that keep per-launch global counters (GEMM round sync, attention
// unit queue, streamed-row pool): distinct streams of a device never share a
// slot, so their concurrent launches cannot disturb each other's counters.
// Returns -1 once a device has handed out all slots (the caller then runs the
// counter-free variant). `kind` separates the kernels' slot spaces.
int stream_slot(void* stream, int kind, int nslots);
void count_launch(int n = 1);

// Encodes a 2-D tiled TMA descriptor with 128-byte swizzle over a row-major
// matrix of `rows` x `cols` elements (cols contiguous, row pitch `ld`
// elements), box = box_rows x box_cols.
afg_status make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                        int elem_bytes, int64_t cols, int64_t rows, int64_t ld,
                        int box_cols, int box_rows,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);
// General tiled descriptor (rank <= 5), dims/strides innermost first,
// strides in bytes for dims 1..rank-1.
afg_status make_tmap(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int rank,
                     const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box, CUtensorMapSwizzle swz);

// im2col descriptor over an NHWC tensor (dims C, W, H, N innermost first);
// lower/upper = {W, H} bounding-box corners, traversal strides sw/sh.
afg_status make_tmap_im2col_4d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                               int64_t C, int64_t W, int64_t H, int64_t N, const int* lower,
                               const int* upper, int sw, int sh, int channels, int pixels,
                               int elem_bytes = 2);

inline int dtype_bytes(afg_dtype t) { return t == AFG_F32 ? 4 : 2; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool valid_dtype(int t) { return t == AFG_F32 || t == AFG_F16 || t == AFG_BF16; }
// AFG_OK iff a compute-capability-10.x device is current (no CPU fallback).
afg_status check_device();


// Sets a kernel's dynamic shared-memory opt-in once per device (the attribute
// is per device; `done` is the call site's own bit set, one bit per device).
template <typename Kern>
inline cudaError_t ensure_smem_optin(std::atomic<uint64_t>& done, Kern kern, int smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// ---- kernel families (each .cu file) ---------------------------------------
afg_status gemm_tc(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                   const void* residual, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                   afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                   cudaStream_t stream);

// Programmatic dependent launch for the persistent kernels (they wait on the
// previous grid with griddepcontrol.wait after their prologue); AFG_PDL=0
// disables it for A/B measurements.
bool pdl_enabled();
afg_status conv_halo(const void* x, const void* w, const float* bias, void* y, int64_t B,
                     int64_t H, int64_t W, int64_t C, int64_t OC, afg_dtype dt, afg_dtype yt,
                     afg_epilogue epi, cudaStream_t stream);
afg_status conv_tc(const void* x, const void* w, const float* bias, void* y, int64_t B,
                   int64_t H, int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                   int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t dh, int64_t dw,
                   int64_t OH, int64_t OW, afg_dtype dt, afg_dtype yt, afg_epilogue epi,
                   cudaStream_t stream);

afg_status gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                     const void* residual, void* C, int64_t ldc, int64_t M, int64_t N,
                     int64_t K, int64_t batch, int64_t sA, int64_t sB, int64_t sC,
                     afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                     cudaStream_t stream);

}  // namespace afg
