timeout 300 python bench.py --workload gemm_i8 --size 8192 --steps 10 --warmup 3 > gpurun_out/bench_gemm_i8_8192.json 2> gpurun_out/bench_gemm_i8.err
timeout 300 python bench.py --workload gemm_i8 --steps 10 --warmup 3 > gpurun_out/bench_gemm_i8.json 2>> gpurun_out/bench_gemm_i8.err
timeout 300 python bench.py --workload gemm_i8 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_gemm_i8_reference.json 2>> gpurun_out/bench_gemm_i8.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gemm_i8.csv python bench.py --workload gemm_i8 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
cat gpurun_out/bench_gemm_i8_8192.json gpurun_out/bench_gemm_i8.json gpurun_out/bench_gemm_i8_reference.json | cut -c1-600; tail -3 gpurun_out/bench_gemm_i8.err
