#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
python scripts/vm_region_probe.py 2048 4096
AFG_NEST_JIT=0 python scripts/vm_region_probe.py 2048 4096
for t in 64 128; do AFG_SIMT_TPB=$t python bench.py --workload gemm_fp32 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('simt_tpb=$t', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
} > gpurun_out/jit.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:nest_jit --clock-control none -c 3 --csv python scripts/vm_region_probe.py 2048 4096 > gpurun_out/jit_ncu.csv 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x >> gpurun_out/jit.txt 2>&1
tail -30 gpurun_out/jit.txt
