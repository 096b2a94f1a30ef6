#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/pool3.txt; : > $o
for t in tests/test_chains_gpu.py tests/test_encoder_gpu.py tests/test_graph_gpu.py; do
timeout 300 python -m pytest $t -q -x -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed|^E " | head -8 >> $o
done
AFG_STREAM_POOL=0 timeout 300 python -m pytest tests/test_encoder_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> $o
cat $o
