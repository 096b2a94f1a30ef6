#!/bin/bash
# A/B of the output-bound short-K GEMM (ResNet 1x1 convs) epilogue configurations
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/shortk.txt; : > $o
echo "== default" >> $o; timeout 200 python scripts/conv1x1_probe.py 2>&1 | grep -v Warn >> $o
echo "== groups4" >> $o; AFG_GEMM_SHORTK_GROUPS=4 timeout 200 python scripts/conv1x1_probe.py 2>&1 | grep -v Warn >> $o
echo "== bn128" >> $o; AFG_GEMM_BN=128 timeout 200 python scripts/conv1x1_probe.py 2>&1 | grep -v Warn >> $o
echo "== early0" >> $o; AFG_EPI_EARLY_TMEM=0 timeout 200 python scripts/conv1x1_probe.py 2>&1 | grep -v Warn >> $o
echo "== notma" >> $o; AFG_GEMM_TMA_STORE=0 timeout 200 python scripts/conv1x1_probe.py 2>&1 | grep -v Warn >> $o
AFG_GEMM_SHORTK_GROUPS=4 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
echo "gemm16384 $(timeout 200 python bench.py --size 16384 --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), d["clocks"])')" >> $o
cat $o
