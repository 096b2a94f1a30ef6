#!/bin/bash
# One GPU session: gemm tests, headline bench, ncu launch list + full capture.
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gemm_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/gemm_tests.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_gemm16k.json 2> gpurun_out/bench_gemm16k.err
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --size 8192 --no-cpu-baseline > gpurun_out/bench_gemm8k.json 2>&1
timeout -s KILL 200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_gemm16k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_gemm16k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
