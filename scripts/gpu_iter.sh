#!/bin/bash
# Iteration run: selected gpu tests, selected bench workloads, optional ncu captures.
#   TESTS="tests/test_x.py ..."  WLS="softmax attention"  NCU="wl:regex:tag ..."
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout -s KILL 900 python -m pytest $TESTS -m gpu -q -p no:cacheprovider -x 2>&1 | tail -25 > gpurun_out/iter_tests.log
fi
for w in $WLS; do
  timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 $BENCH_EXTRA > gpurun_out/iter_$w.json 2> gpurun_out/iter_$w.err
  python3 -c "import json;d=json.load(open('gpurun_out/iter_$w.json'));r=d['roofline'];print('$w', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'kernel_frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/iter_summary.txt 2>&1 || tail -3 gpurun_out/iter_$w.err >> gpurun_out/iter_summary.txt
done
for spec in $NCU; do
  IFS=: read w rx tag <<< "$spec"
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_$tag.log 2>&1
done
echo done
