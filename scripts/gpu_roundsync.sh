#!/bin/bash
# A/B: round-synchronised producers (AFG_GEMM_ROUND_SYNC) on the 16384^3 / 8192^3 GEMMs
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/roundsync.txt; : > $o
for rs in 0 1 0 1; do
  for n in 16384 8192; do
    echo "sync=$rs n=$n $(AFG_GEMM_ROUND_SYNC=$rs timeout 200 python bench.py --size $n --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), d["clocks"])')" >> $o
  done
done
for rs in 0 1; do
  AFG_GEMM_ROUND_SYNC=$rs timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tc -s 3 -c 1 python bench.py --size 16384 --only --no-cpu-baseline --steps 2 --warmup 3 2>&1 | grep -E "dram__|duration|hit_rate|tensor" | sed "s/^/sync=$rs /" >> $o
done
python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
AFG_GEMM_ROUND_SYNC=1 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
cat $o
