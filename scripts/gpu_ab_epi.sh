#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for rep in 1 2; do
for e in 0 1; do
  for n in 16384 8192 4096; do AFG_EPI_EARLY_TMEM=$e python bench.py --workload gemm_bf16 --size $n --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early=$e gemm $n', round(d['value'],1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
  for w in resnet50_convs bert_layer; do AFG_EPI_EARLY_TMEM=$e python bench.py --workload $w --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early=$e $w', round(d['value'],1), d['roofline'].get('frac_of_op_floor'))"; done
done
done
} > gpurun_out/ab_epi.txt 2>&1
cat gpurun_out/ab_epi.txt
for t in 128 256 64; do AFG_SIMT_TPB=$t python bench.py --workload gemm_fp32 --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('simt_tpb=$t', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done >> gpurun_out/ab_epi.txt 2>&1
AFG_SIMT_TPB=256 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider -k "fp32" >> gpurun_out/ab_epi.txt 2>&1
tail -4 gpurun_out/ab_epi.txt
