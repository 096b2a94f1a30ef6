#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
python scripts/gemm_shape_time.py 2048x2048x2048:gelu:kn 2048x2048x4096:gelu:kn 2048x2048x8192:gelu:kn 2048x2048x16384:gelu:kn 2048x2048x2048:none:kn 4096x2048x2048:gelu:kn 2048x4096x2048:gelu:kn
AFG_GEMM_BN=128 python scripts/gemm_shape_time.py 2048x2048x2048:gelu:kn
} > gpurun_out/gemm_shapes.txt 2>&1
cat gpurun_out/gemm_shapes.txt
