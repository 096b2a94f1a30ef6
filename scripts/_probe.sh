timeout 300 python -m pytest tests/test_gemm_i8_gpu.py tests/test_graph_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
for n in 16384 8192; do
timeout 300 python bench.py --workload gemm_i8 --size $n --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('n=$n', round(d['value'],1), round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['frac'],3))"
done
