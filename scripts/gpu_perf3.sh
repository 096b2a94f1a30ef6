#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for w in layernorm softmax; do timeout 300 python bench.py --workload $w --only --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
timeout 300 python bench.py --workload bert_layer --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bert', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_of_op_floor'))"
} > gpurun_out/perf3.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:stream_rows --clock-control none -s 5 -c 2 --csv python bench.py --workload layernorm --only --steps 5 --no-cpu-baseline --no-graph > gpurun_out/ln_ncu2.csv 2>/dev/null
timeout 600 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py -q -p no:cacheprovider >> gpurun_out/perf3.txt 2>&1
cat gpurun_out/perf3.txt | tail -20
