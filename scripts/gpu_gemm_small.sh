#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/gemm_small.txt; : > $o
timeout 200 python scripts/gemm_small_probe.py 2048 4096 >> $o 2>&1
PROBE_TAG=pair AFG_GEMM_PAIR=2 timeout 200 python scripts/gemm_small_probe.py 2048 >> $o 2>&1
PROBE_TAG=bn128 AFG_GEMM_BN=128 timeout 200 python scripts/gemm_small_probe.py 2048 >> $o 2>&1
PROBE_TAG=noflush AFG_BENCH_NO_FLUSH=1 timeout 200 python scripts/gemm_small_probe.py 2048 >> $o 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max --clock-control none -k regex:gemm_tc -c 6 python scripts/gemm_small_probe.py 2048 2>&1 | grep -E "gemm_tc|duration|cycles" | head -24 >> $o
cat $o
