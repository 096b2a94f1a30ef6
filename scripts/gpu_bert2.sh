#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/bert2.txt; : > $o
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_encoder_gpu.py -q -p no:cacheprovider 2>&1 | tail -1 >> $o
timeout 300 python scripts/bert_gemm_probe.py >> $o 2>&1
for rep in 1 2; do
echo "bert $(timeout 200 python bench.py --workload bert_layer --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"].get("frac_of_op_floor",0),3), round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["reasons"])')" >> $o
done
cat $o
