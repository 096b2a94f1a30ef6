#!/bin/bash
# 16384^3 GEMM: DRAM bytes per launch vs the raster group (AFG_GEMM_GROUP_M, pair-tile rows)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for g in 4 8 16 32; do
  AFG_GEMM_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:gemm_tc_kernel -s 3 -c 1 --clock-control none --csv python bench.py --workload gemm_bf16 --size 16384 --only --steps 1 --no-graph --no-cpu-baseline 2>/dev/null | grep gemm_tc | awk -F'","' -v g=$g '{print "group " g, $(NF-2), $NF}'
  AFG_GEMM_GROUP_M=$g python bench.py --workload gemm_bf16 --size 16384 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('group $g time', round(d['value'],1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done > gpurun_out/gemm_traffic.txt 2>&1
cat gpurun_out/gemm_traffic.txt
