#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/dyn64.txt; : > $o
for dyn in 1 0; do for d in 0 3; do
  AFG_ATTN_DYN=$dyn AFG_ATTN_DEBUG=$d python scripts/attn_shape_probe.py 64 12 512 64 bf16 0 | sed "s/^/dyn=$dyn /" >> $o 2>&1
done; done
cat $o
