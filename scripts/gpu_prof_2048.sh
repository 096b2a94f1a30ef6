#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/prof/gemm2048 python bench.py --workload gemm_bf16 --size 2048 --only --steps 2 --no-graph --no-cpu-baseline > gpurun_out/prof/g2048.log 2>&1
ncu -i gpurun_out/prof/gemm2048.ncu-rep --page raw --csv > gpurun_out/prof/gemm2048_raw.csv 2>/dev/null
ncu -i gpurun_out/prof/gemm2048.ncu-rep --page details --csv > gpurun_out/prof/gemm2048_details.csv 2>/dev/null
rm -f gpurun_out/prof/*.ncu-rep
ls -la gpurun_out/prof
