#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; o=gpurun_out/view.txt; : > $o
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_graph_scale_gpu.py tests/test_sharded_graph_gpu.py tests/test_reference_suites_gpu.py tests/test_reference_swap_gpu.py tests/test_spec_grids_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|passed|failed" >> $o
AFG_GRAPH_TIMING=1 python scripts/graph_api_probe.py 4096 >> $o 2>&1
python -c "import __graft_entry__ as g; g.smoke()" >> $o 2>&1
cat $o
