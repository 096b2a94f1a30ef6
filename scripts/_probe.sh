for d in 2 1 2 1; do for n in 2048 3072; do
AFG_GEMM_PAIR=$d timeout 300 python bench.py --workload gemm_bf16 --size $n --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('PAIR=$d n=$n', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us')"
done; done
