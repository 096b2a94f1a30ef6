#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -4
for w in softmax layernorm bert_layer; do
  timeout -s KILL 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3_$w.json 2>&1
  python3 -c "import json;d=json.load(open('gpurun_out/bench3_$w.json'));print('$w', round(d['value'],1), d['unit'], 'kernel', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))"
done
