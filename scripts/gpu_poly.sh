#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/poly.txt; : > $o
for rep in 1 2; do for pp in 0x12 0x02 0x00 0x11 0x52 0x55; do for wl in attention attention_causal bert_layer; do
  echo "$pp $wl $(AFG_LIB_PATH=variants/libafg_poly$pp.so timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')" >> $o
done; done; done
AFG_LIB_PATH=variants/libafg_poly0x55.so timeout 300 python -m pytest tests/test_attention_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
cat $o
