#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_attention_gpu.py tests/test_encoder_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -4
for w in attention attention_causal bert_layer; do
  timeout -s KILL 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_$w.json 2>&1
  python3 -c "import json;d=json.load(open('gpurun_out/bench5_$w.json'));print('$w', round(d['value'],1), d['unit'], 'kernel frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:stream_rows -s 3 -c 1 -o gpurun_out/prof_ln python bench.py --workload layernorm --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:stream_rows -s 3 -c 1 -o gpurun_out/prof_sm python bench.py --workload softmax --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
