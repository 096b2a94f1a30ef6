#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof_d64
for d in 0 3; do
AFG_ATTN_DEBUG=$d timeout 400 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_d64/d64_dbg$d -f python scripts/attn_shape_probe.py 64 12 512 64 bf16 0 > /dev/null 2>&1
f=gpurun_out/prof_d64/d64_dbg$d.ncu-rep
ncu -i $f --page raw --csv > gpurun_out/prof_d64/d64_dbg${d}_raw.csv 2>/dev/null
ncu -i $f --page details --csv > gpurun_out/prof_d64/d64_dbg${d}_details.csv 2>/dev/null
ncu -i $f --page source --csv --print-source sass > gpurun_out/prof_d64/d64_dbg${d}_sass.csv 2>/dev/null
gzip -f gpurun_out/prof_d64/d64_dbg${d}_sass.csv gpurun_out/prof_d64/d64_dbg${d}_raw.csv; rm -f $f
done
ls gpurun_out/prof_d64
