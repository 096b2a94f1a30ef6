#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/skip2.txt; : > $o
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -5 >> $o
for rep in 1 2; do for v in old new; do
  L=variants/libafg_$v.so
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 8 16 2048 128 f16 1)" >> $o
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 8 16 2048 128 f16 0)" >> $o
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
done; done
cat $o
