#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/halo2.txt; : > $o
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py tests/test_spec_grids_gpu.py tests/test_graph_scale_gpu.py -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -5 >> $o
for s in "256 56 64 64 3 1" "256 28 128 128 3 1" "256 14 256 256 3 1" "256 7 512 512 3 1"; do python scripts/conv_shape_probe.py $s >> $o 2>&1; done
for rep in 1 2; do echo "resnet $(timeout 300 python bench.py --workload resnet50_convs --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"].get("frac_of_op_floor",0),3), round(d["ms_per_step"]*1e3,1), "us")')" >> $o; done
cat $o
