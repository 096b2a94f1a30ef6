#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for kb in 216 192; do AFG_LN_SMEM_KB=$kb python bench.py --workload layernorm --only --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ln kb=$kb', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
for w in softmax bert_layer; do python bench.py --workload $w --only --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
} > gpurun_out/ln.txt 2>&1
timeout 600 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py tests/test_reference_swap_gpu.py -q -p no:cacheprovider >> gpurun_out/ln.txt 2>&1
oracle/_ref/check_lowering_gpu tests/golden/check_lowering_cases.json > gpurun_out/check_lowering.txt 2>&1
tail -20 gpurun_out/ln.txt
