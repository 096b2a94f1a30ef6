#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/mask.txt; : > $o
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -5 >> $o
for rep in 1 2; do for wl in attention attention_causal; do
  echo "$wl $(timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done; done
cat $o
