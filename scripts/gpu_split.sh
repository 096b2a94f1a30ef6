#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/split.txt; : > $o
AFG_LIB_PATH=variants/libafg_split.so timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -5 >> $o
for rep in 1 2; do for v in base split; do for wl in attention attention_causal bert_layer; do
  echo "$v $wl $(AFG_LIB_PATH=variants/libafg_$v.so timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done; done; done
cat $o
