#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/shortk2.txt; : > $o
for s in "50176 256 1024" "200704 512 256" "50176 1024 256" "12544 512 2048" "12544 2048 512" "50176 1024 512"; do
  for cfg in "X=0" "AFG_GEMM_SHORTK_MAXK=4096" "AFG_GEMM_BN=128" "AFG_EPI_EARLY_TMEM=0" "AFG_EPI_EARLY_TMEM=1" "AFG_GEMM_PAIR=0" "AFG_GEMM_PAIR=2"; do
    echo "[$cfg] $(env $cfg python scripts/gemm_shape_probe.py $s 2>&1 | tail -1)" >> $o
  done
done
cat $o
