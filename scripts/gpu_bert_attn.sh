#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/bert_attn.txt; : > $o
for d in 0 1 2 3; do AFG_ATTN_DEBUG=$d python scripts/attn_shape_probe.py 64 12 512 64 bf16 0 >> $o 2>&1; done
for d in 0 1 2 3; do AFG_ATTN_DEBUG=$d python scripts/attn_shape_probe.py 16 12 2048 64 bf16 0 >> $o 2>&1; done
cat $o
