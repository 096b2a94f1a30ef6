#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/bert_gemm.txt; : > $o
timeout 300 python scripts/bert_gemm_probe.py >> $o 2>&1
echo "== 2 epi groups" >> $o; AFG_GEMM_EPI_GROUPS=2 timeout 300 python scripts/bert_gemm_probe.py >> $o 2>&1
echo "== no pair" >> $o; AFG_GEMM_PAIR=0 timeout 300 python scripts/bert_gemm_probe.py >> $o 2>&1
cat $o
