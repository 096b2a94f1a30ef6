#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof2048; o=gpurun_out/prof2048/summary.txt; : > $o
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,lts__t_sector_hit_rate.pct"
for cfg in "X=0" "AFG_GEMM_PAIR=2" "AFG_GEMM_BN=256"; do
  echo "== $cfg" >> $o
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_tc -s 8 -c 2 python scripts/gemm_small_probe.py 2048 2>&1 | grep -E "gemm_tc_kernel<|duration|tensor|lts__|dram__|xbar|cycles" | sed 's/^ *//' | cut -c1-150 >> $o
done
cat $o
