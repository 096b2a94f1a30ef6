#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -6
for w in gemm_bf16 resnet50_convs bert_layer; do
  timeout -s KILL 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench4_$w.json 2>&1
  python3 -c "import json;d=json.load(open('gpurun_out/bench4_$w.json'));print('$w', round(d['value'],1), d['unit'], 'kernel', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))"
done
timeout -s KILL 200 python bench.py --workload gemm_bf16 --size 8192 --steps 10 --warmup 3 --no-cpu-baseline | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('gemm8k', round(d['value'],1))"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file gpurun_out/launches_resnet3.csv python bench.py --workload resnet50_convs --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_bert2.csv python bench.py --workload bert_layer --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
