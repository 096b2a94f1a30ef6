#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/cps.txt; : > $o
v() { timeout 200 python bench.py "$@" --only --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us")'; }
for rep in 1 2; do for c in 1 2; do
  echo "cps=$c layernorm $(AFG_STREAM_CPS=$c v --workload layernorm)  softmax $(AFG_STREAM_CPS=$c v --workload softmax)" >> $o
done; done
AFG_STREAM_CPS=2 timeout 600 python -m pytest tests/test_chains_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
cat $o
