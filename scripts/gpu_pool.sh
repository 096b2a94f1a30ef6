#!/bin/bash
# stream kernels (softmax / layernorm) with the dynamic tail pool: parity + A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/pool.txt; : > $o
timeout 600 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
AFG_STREAM_POOL=4 timeout 600 python -m pytest tests/test_chains_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
for rep in 1 2; do for p in 0 16 8 4; do for wl in layernorm softmax; do
  echo "$wl pool=$p $(AFG_STREAM_POOL=$p timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us", d["clocks"]["reasons"])')" >> $o
done; done; done
AFG_STREAM_POOL=16 timeout 300 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.avg,gpu__time_duration.sum --clock-control none -k regex:stream_rows -s 5 -c 1 python bench.py --workload layernorm --only --steps 1 --warmup 5 --no-cpu-baseline --no-graph 2>&1 | grep -E "sm__|duration" >> $o
cat $o
