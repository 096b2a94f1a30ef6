#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/bert_attn.txt; : > $o
for d in 0 1 2 3; do AFG_ATTN_DEBUG=$d python scripts/attn_shape_probe.py 64 12 512 64 bf16 0 >> $o 2>&1; done
for d in 0 1 2 3; do AFG_ATTN_DEBUG=$d python scripts/attn_shape_probe.py 8 16 2048 128 f16 0 >> $o 2>&1; done
cat $o
