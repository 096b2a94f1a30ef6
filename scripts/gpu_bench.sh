#!/bin/bash
# gpurun helper: the default bench line (headline + workloads sub-dict) and,
# optionally, the reference arm; outputs under gpurun_out/
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$WITH_REF" ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
fi
tail -c 3000 gpurun_out/bench.json
