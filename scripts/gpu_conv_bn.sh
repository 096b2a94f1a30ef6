#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/conv_bn.txt; : > $o
for s in "256 7 512 512 3 1" "256 14 512 512 3 2" "256 28 256 256 3 2" "256 56 128 128 3 2" "256 14 1024 2048 1 2" "256 28 512 1024 1 2" "256 56 256 512 1 2"; do
  for cfg in "X=0" "AFG_CONV_BN=128" "AFG_GEMM_PAIR=0" "AFG_GEMM_PAIR=2"; do
    env $cfg python scripts/conv_shape_probe.py $s >> $o 2>&1
  done
done
cat $o
