#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof_k64
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_k64/k64 -f python scripts/gemm_shape_probe.py 802816 64 256 > /dev/null 2>&1
f=gpurun_out/prof_k64/k64.ncu-rep
ncu -i $f --page raw --csv > gpurun_out/prof_k64/k64_raw.csv 2>/dev/null
ncu -i $f --page details --csv > gpurun_out/prof_k64/k64_details.csv 2>/dev/null
ncu -i $f --page source --csv --print-source sass > gpurun_out/prof_k64/k64_sass.csv 2>/dev/null
gzip -f gpurun_out/prof_k64/k64_sass.csv gpurun_out/prof_k64/k64_raw.csv; rm -f $f
python scripts/gemm_shape_probe.py 802816 64 256
