#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof1x1; o=gpurun_out/prof1x1/times.txt; : > $o
for s in "50176 256 1024" "802816 64 256" "200704 128 512" "12544 512 2048"; do
  python scripts/gemm_shape_probe.py $s >> $o 2>&1
  AFG_GEMM_SHORTK_GROUPS=2 python scripts/gemm_shape_probe.py $s | sed 's/^/g2 /' >> $o 2>&1
done
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 5 -c 1 -o gpurun_out/prof1x1/g50176_256_1024 -f python scripts/gemm_shape_probe.py 50176 256 1024 > /dev/null 2>&1
f=gpurun_out/prof1x1/g50176_256_1024.ncu-rep
ncu -i $f --page raw --csv > gpurun_out/prof1x1/g50176_256_1024_raw.csv 2>/dev/null
ncu -i $f --page details --csv > gpurun_out/prof1x1/g50176_256_1024_details.csv 2>/dev/null
ncu -i $f --page source --csv --print-source sass > gpurun_out/prof1x1/g50176_256_1024_sass.csv 2>/dev/null
gzip -f gpurun_out/prof1x1/*_sass.csv gpurun_out/prof1x1/*_raw.csv; rm -f $f
cat $o
