#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for f in 1 0; do AFG_SIMT_FAST=$f python bench.py --workload gemm_fp32 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('simt_fast=$f', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
python bench.py --workload layernorm --only --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layernorm', d['value'], d['ms_per_step'], d['roofline']['frac'])"
} > gpurun_out/perf2.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:stream_rows --clock-control none -s 5 -c 3 --csv python bench.py --workload layernorm --only --steps 5 --no-cpu-baseline --no-graph > gpurun_out/ln_ncu.csv 2>/dev/null
timeout 900 python -m pytest tests/test_spec_grids_gpu.py tests/test_graph_gpu.py tests/test_graph_scale_gpu.py tests/test_gemm_gpu.py -q -p no:cacheprovider >> gpurun_out/perf2.txt 2>&1
cat gpurun_out/perf2.txt | tail -40
