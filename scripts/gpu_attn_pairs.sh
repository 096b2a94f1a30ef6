#!/bin/bash
# attention: pair-register S loads + dynamic queue: parity + bench + decomposition
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/attn_pairs.txt; : > $o
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
for rep in 1 2; do for wl in attention attention_causal bert_layer; do
  echo "$wl $(timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["reasons"])')" >> $o
done; done
for d in 1 2 3; do
  echo "attention dbg=$d $(AFG_ATTN_DEBUG=$d timeout 200 python bench.py --workload attention --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done
cat $o
