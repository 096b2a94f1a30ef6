#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for kb in 192 96 48; do AFG_LN_SMEM_KB=$kb python bench.py --workload layernorm --only --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ln kb=$kb', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
AFG_BENCH_NO_FLUSH=1 python bench.py --workload layernorm --only --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ln noflush (L2-warm, diagnostic)', d['value'], d['ms_per_step'], d['roofline']['frac'])"
python bench.py --workload gemm_bf16 --size 2048 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gemm2048', d['value'], d['roofline']['frac'])"
} > gpurun_out/perf5.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider >> gpurun_out/perf5.txt 2>&1
bash scripts/gpu_sanitize.sh >> gpurun_out/perf5.txt 2>&1
tail -40 gpurun_out/perf5.txt
