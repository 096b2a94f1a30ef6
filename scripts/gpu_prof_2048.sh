#!/bin/bash
# ncu --set full of the 2048^3 GEMM (flushed L2, as in the bench), NONE and GELU epilogues
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof2048
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 8 -c 1 \
  -o gpurun_out/prof2048/g2048_none -f python scripts/gemm_small_probe.py 2048 > gpurun_out/prof2048/log.txt 2>&1
for f in gpurun_out/prof2048/*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null
done
ls -la gpurun_out/prof2048
