#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/rpre.txt; : > $o
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -5 >> $o
python scripts/bert_gemm_probe.py >> $o 2>&1
for rep in 1 2; do echo "bert $(timeout 300 python bench.py --workload bert_layer --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"].get("frac_of_op_floor",0),3), round(d["ms_per_step"]*1e3,1), "us")')" >> $o; done
cat $o
