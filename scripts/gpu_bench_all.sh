#!/bin/bash
mkdir -p gpurun_out
for w in gemm_bf16 gemm_fp32 attention attention_causal resnet50_convs bert_layer softmax layernorm; do
  timeout -s KILL 240 python bench.py --workload $w --steps 10 --warmup 3 ${EXTRA} > gpurun_out/bench6_$w.json 2> gpurun_out/bench6_$w.err
  python3 -c "import json;d=json.load(open('gpurun_out/bench6_$w.json'));print('$w', round(d['value'],1), d['unit'], 'step_ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done
