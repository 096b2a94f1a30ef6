#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/lnrows.txt; : > $o
for rep in 1 2; do for r in 2 4 1; do
  echo "rows=$r $(AFG_LIB_PATH=variants/libafg_ln$r.so timeout 200 python bench.py --workload layernorm --only --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us")')" >> $o
done; done
AFG_LIB_PATH=variants/libafg_ln4.so timeout 600 python -m pytest tests/test_chains_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
cat $o
