#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/sanitize
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/sanitize/racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize/racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/sanitize/synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize/synccheck.txt
tail -4 gpurun_out/sanitize/racecheck.txt gpurun_out/sanitize/synccheck.txt
timeout 600 python -m pytest tests/test_chains_gpu.py tests/test_encoder_gpu.py -q -p no:cacheprovider 2>&1 | tail -1
for wl in layernorm softmax; do timeout 200 python bench.py --workload $wl --only --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["roofline"]["frac"],3))'; done
