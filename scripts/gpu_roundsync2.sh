#!/bin/bash
# round sync default-on: parity, ResNet A/B, 1x1 store-path probe
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/roundsync2.txt; : > $o
python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_graph_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> $o
for rs in 0 1 0 1; do
  echo "sync=$rs resnet $(AFG_GEMM_ROUND_SYNC=$rs timeout 300 python bench.py --workload resnet50_convs --only --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"].get("frac_of_op_floor",0),3), d["clocks"]["reasons"])')" >> $o
done
timeout 300 python scripts/conv1x1_probe.py >> $o 2>&1
cat $o
