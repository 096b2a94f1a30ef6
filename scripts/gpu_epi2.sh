#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/epi2.txt; : > $o
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py tests/test_splitk_gpu.py tests/test_spec_grids_gpu.py -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" | head -5 >> $o
for s in "802816 64 256" "200704 128 512" "50176 256 1024" "12544 512 2048"; do python scripts/gemm_shape_probe.py $s >> $o 2>&1; done
python scripts/bert_gemm_probe.py >> $o 2>&1
for wl in resnet50_convs bert_layer; do
  echo "$wl $(timeout 300 python bench.py --workload $wl --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"].get("frac_of_op_floor",0),3), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done
echo "gemm16384 $(timeout 200 python bench.py --size 16384 --only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1))')" >> $o
cat $o
