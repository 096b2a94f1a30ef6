O=gpurun_out/i8
mkdir -p $O
timeout 300 python bench.py --workload gemm_i8 --steps 10 --warmup 3 > $O/bench_gemm_i8.json 2> $O/err.txt
timeout 300 python bench.py --workload gemm_i8 --size 8192 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gemm_i8_8192.json 2>> $O/err.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gemm_i8.csv python bench.py --workload gemm_i8 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 3 -c 1 -o $O/full_gemm_i8_16384 python bench.py --workload gemm_i8 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/full.log 2>&1
ncu -i $O/full_gemm_i8_16384.ncu-rep --page raw --csv > $O/full_gemm_i8_16384_raw.csv 2>/dev/null
ncu -i $O/full_gemm_i8_16384.ncu-rep --page details --csv > $O/full_gemm_i8_16384_details.csv 2>/dev/null
ncu -i $O/full_gemm_i8_16384.ncu-rep --page source --csv --print-source sass > $O/full_gemm_i8_16384_sass.csv 2>/dev/null
gzip -f $O/full_gemm_i8_16384_sass.csv; rm -f $O/full_gemm_i8_16384.ncu-rep
cut -c1-300 $O/bench_gemm_i8.json
