#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for w in resnet50_convs bert_layer; do python bench.py --workload $w --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_of_op_floor'))"; done
for n in 4096 16384; do python bench.py --workload gemm_bf16 --size $n --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gemm $n', d['value'], d['roofline']['frac'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum -k regex:"gemm_tc_kernel|conv_halo_kernel" -c 53 --clock-control none --csv python bench.py --workload resnet50_convs --only --steps 1 --warmup 3 --no-graph --no-cpu-baseline > gpurun_out/resnet_launches.csv 2>/dev/null
python scripts/conv_layers.py gpurun_out/resnet_launches.csv 2>&1 | tail -26
} > gpurun_out/epi.txt 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_encoder_gpu.py tests/test_graph_scale_gpu.py tests/test_spec_grids_gpu.py -q -p no:cacheprovider -x >> gpurun_out/epi.txt 2>&1
tail -45 gpurun_out/epi.txt
