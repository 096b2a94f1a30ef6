#!/bin/bash
mkdir -p gpurun_out
for cfg in "1 2 128 128 0" "1 2 256 64 0" "1 1 384 128 0" "1 2 256 128 1" "1 2 200 128 0" "2 2 512 64 1" "1 1 130 64 1"; do
  timeout -s KILL 30 python scripts/attn_probe.py $cfg 2>&1 | tail -2
done
timeout -s KILL 240 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -4
for w in attention attention_causal bert_layer; do
  timeout -s KILL 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench2_$w.json 2>&1
  python3 -c "import json;d=json.load(open('gpurun_out/bench2_$w.json'));print('$w', round(d['value'],1), d['unit'], 'kernel frac', round(d['roofline']['frac'],3))"
done
