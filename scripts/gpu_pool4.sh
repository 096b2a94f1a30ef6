#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/pool4.txt; : > $o
timeout 900 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -20 >> $o
for rep in 1 2; do for p in -1 0 4; do for wl in layernorm softmax; do
  [ "$p" = "-1" ] && unset AFG_STREAM_POOL || export AFG_STREAM_POOL=$p
  echo "$wl pool=$p $(timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us", d["clocks"]["reasons"])')" >> $o
done; done; done
cat $o
