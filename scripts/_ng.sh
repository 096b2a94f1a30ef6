for i in 1 2; do for g in 2 4; do
AFG_GEMM_EPI_GROUPS=$g timeout 300 python bench.py --workload bert_layer --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('NG=$g', d['value'], d['ms_per_step'], d['clocks'])"
done; done
