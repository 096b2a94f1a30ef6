#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/misc_ab.txt; : > $o
v() { timeout 200 python bench.py "$@" --only --no-cpu-baseline --steps 30 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us")'; }
for kb in 0 160 208 220; do
  if [ $kb = 0 ]; then unset AFG_LN_SMEM_KB; else export AFG_LN_SMEM_KB=$kb; fi
  echo "layernorm smem=$kb $(v --workload layernorm) $(v --workload layernorm)" >> $o
done
unset AFG_LN_SMEM_KB
for cfg in "" "AFG_GEMM_BN=64" "AFG_GEMM_BN=256" "AFG_GEMM_PAIR=2" "AFG_EPI_EARLY_TMEM=0"; do
  echo "gemm2048 [$cfg] $(env $cfg bash -c 'timeout 200 python bench.py --size 2048 --only --no-cpu-baseline --steps 30 --warmup 3 2>/dev/null' | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3), round(d["ms_per_step"]*1e3,2), "us")')" >> $o
done
cat $o
