#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_encoder_gpu.py tests/test_attention_gpu.py -q -m gpu -p no:cacheprovider -s 2>&1 | tail -15 > gpurun_out/enc_tests.log
for w in attention attention_causal resnet50_convs bert_layer softmax layernorm gemm_fp32; do
  timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_bert.csv python bench.py --workload bert_layer --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file gpurun_out/launches_resnet.csv python bench.py --workload resnet50_convs --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_attn python bench.py --workload attention --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
timeout -s KILL 400 ncu --set full --clock-control none -k regex:softmax_warp -s 3 -c 1 -o gpurun_out/prof_softmax python bench.py --workload softmax --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_softmax.log 2>&1
echo done
