#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/desc.txt; : > $o
for rep in 1 2; do for v in d0 d1; do
  L=variants/libafg_$v.so
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
  echo "$v $(AFG_LIB_PATH=$L AFG_ATTN_DEBUG=3 python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 8 16 2048 128 f16 0)" >> $o
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 8 16 2048 128 f16 1)" >> $o
done; done
AFG_LIB_PATH=variants/libafg_d1.so timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
cat $o
