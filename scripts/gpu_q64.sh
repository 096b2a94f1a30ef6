#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/q64.txt; : > $o
for rep in 1 2; do for v in q2 q1; do
  L=variants/libafg_$v.so
  echo "$v $(AFG_LIB_PATH=$L python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
  echo "$v $(AFG_LIB_PATH=$L AFG_ATTN_DEBUG=3 python scripts/attn_shape_probe.py 64 12 512 64 bf16 0)" >> $o
done; done
cat $o
