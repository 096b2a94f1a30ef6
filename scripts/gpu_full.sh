#!/bin/bash
# Full GPU check: smoke, pytest -m gpu, every bench workload, default-bench launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
for w in gemm_bf16 gemm_fp32 attention attention_causal resnet50_convs bert_layer softmax layernorm; do
  timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout -s KILL 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo done
