#!/bin/bash
# attention decomposition: AFG_ATTN_DEBUG 0 (full), 1 (no softmax math), 2 (no MMAs), 3 (MMAs only)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/attn_dbg.txt; : > $o
for wl in attention attention_causal; do
for d in 0 1 2 3; do
  echo "$wl dbg=$d $(AFG_ATTN_DEBUG=$d timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["reasons"])')" >> $o
done; done
cat $o
