#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/attn_dyn2.txt; : > $o
for rep in 1 2; do for cfg in "0 0" "1 16" "1 8" "1 32"; do set -- $cfg
  echo "causal dyn=$1 hg=$2 $(AFG_ATTN_HEAD_GROUP=$2 AFG_ATTN_DYN=$1 timeout 200 python bench.py --workload attention_causal --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["reasons"])')" >> $o
done; done
cat $o
