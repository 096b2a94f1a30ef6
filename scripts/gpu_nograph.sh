#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/nograph.txt; : > $o
v() { timeout 200 python bench.py "$@" --only --no-cpu-baseline --steps 30 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us")'; }
for rep in 1 2; do
for a in "--size 2048" "--size 4096" "--workload layernorm" "--workload softmax" "--workload attention_causal"; do
  echo "$a graph: $(v $a)   nograph: $(v $a --no-graph)" >> $o
done; done
cat $o
