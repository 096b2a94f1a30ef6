#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/slots.txt; : > $o
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_chains_gpu.py tests/test_gemm_gpu.py tests/test_encoder_gpu.py tests/test_splitk_gpu.py tests/test_sharded_graph_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" >> $o
for wl in attention_causal softmax; do
echo "$wl $(timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3))')" >> $o
done
echo "gemm16384 $(timeout 200 python bench.py --size 16384 --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1))')" >> $o
cat $o
