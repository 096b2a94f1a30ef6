#!/bin/bash
# causal attention: head-group size sweep (time + ncu DRAM bytes per launch)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for hg in 8 16 32 64 128; do
  AFG_ATTN_HEAD_GROUP=$hg python scripts/attn_time.py 8 16 2048 128 2>&1 | sed "s/^/hg=$hg /"
done > gpurun_out/attn_sweep.txt
python scripts/attn_time.py 64 12 512 64 >> gpurun_out/attn_sweep.txt 2>&1
for hg in 16 32 128; do
  AFG_ATTN_HEAD_GROUP=$hg timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:attn_fwd --clock-control none -c 4 --csv python scripts/attn_time.py 8 16 2048 128 \
    > gpurun_out/attn_ncu_hg$hg.csv 2>/dev/null
done
cat gpurun_out/attn_sweep.txt
