#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/obuf.txt; : > $o
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -5 >> $o
for rep in 1 2; do for lib in variants/libafg_base.so paper_2603_06731_b200/libafg.so; do
  echo "$lib $(AFG_LIB_PATH=$lib python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
  echo "$lib $(AFG_LIB_PATH=$lib python scripts/attn_shape_probe.py 8 16 2048 128 f16 1)" >> $o
  echo "$lib bert $(AFG_LIB_PATH=$lib timeout 200 python bench.py --workload bert_layer --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done; done
AFG_ATTN_DEBUG=3 python scripts/attn_shape_probe.py 64 12 512 64 bf16 0 >> $o
cat $o
