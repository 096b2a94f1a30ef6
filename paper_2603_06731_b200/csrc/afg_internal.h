// afg_internal.h - host-side plumbing shared by the kernels' launchers and the
// C ABI (api.cpp): status/error reporting, device properties, TMA descriptor
// encoding, launch accounting, and the internal per-family entry points.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/afg.h"

namespace afg {

// Sets the thread-local error message and returns `st`.
afg_status set_error(afg_status st, const char* fmt, ...);
// AFG_OK for cudaSuccess, else AFG_ERR_CUDA with the CUDA error text.
afg_status cuda_status(cudaError_t e, const char* what);

int num_sms();              // SM count of the current device
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

inline int dtype_bytes(afg_dtype t) { return t == AFG_F32 ? 4 : 2; }

// ---- kernel families (each .cu file) ---------------------------------------
afg_status gemm_tc(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                   const void* residual, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                   afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                   cudaStream_t stream);

afg_status gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                     const void* residual, void* C, int64_t ldc, int64_t M, int64_t N,
                     int64_t K, int64_t batch, int64_t sA, int64_t sB, int64_t sC,
                     afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                     cudaStream_t stream);

}  // namespace afg
