#!/bin/bash
# dynamic attention unit queue: parity + A/B + DRAM bytes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/attn_dyn.txt; : > $o
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
for d in 0 1 0 1; do for wl in attention attention_causal bert_layer; do
  echo "$wl dyn=$d $(AFG_ATTN_DYN=$d timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["reasons"])')" >> $o
done; done
for d in 0 1; do for hg in 0 16 64; do
AFG_ATTN_HEAD_GROUP=$hg AFG_ATTN_DYN=$d timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:attn_fwd -s 3 -c 1 python bench.py --workload attention_causal --only --steps 1 --warmup 3 --no-cpu-baseline --no-graph 2>&1 | grep -E "dram__|duration" | sed "s/^/dyn=$d hg=$hg /" >> $o
done; done
cat $o
