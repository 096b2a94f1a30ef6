#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for sc in 0 1; do AFG_ATTN_SCHED=$sc python scripts/attn_time.py 8 16 2048 128 2>&1 | sed "s/^/sched=$sc /"; done
AFG_ATTN_SCHED=1 python scripts/attn_time.py 64 12 512 64 2>&1 | sed "s/^/sched=1 /"
AFG_ATTN_SCHED=0 python scripts/attn_time.py 64 12 512 64 2>&1 | sed "s/^/sched=0 /"
for f in 1 0; do AFG_SIMT_FAST=$f python bench.py --workload gemm_fp32 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('simt_fast=$f', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
} > gpurun_out/perf1.txt 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:attn_fwd --clock-control none -s 3 -c 2 --csv python scripts/attn_time.py 8 16 2048 128 > gpurun_out/attn_ncu_sched.csv 2>/dev/null
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_gemm_gpu.py tests/test_graph_gpu.py -q -x -p no:cacheprovider >> gpurun_out/perf1.txt 2>&1
cat gpurun_out/perf1.txt
