#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
oracle/_ref/check_lowering_gpu tests/golden/check_lowering_cases.json > gpurun_out/check_lowering.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for w in layernorm softmax; do python bench.py --workload $w --only --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log; grep -E "FAIL|SKIP|failure" gpurun_out/check_lowering.txt
