#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:nest_jit --clock-control none -c 2 --csv python scripts/vm_region_probe.py 2048 4096 2>/dev/null | grep nest_jit | awk -F'","' '{print $(NF-2), $NF}' > gpurun_out/jit2.txt
timeout 1200 python -m pytest tests/test_graph_gpu.py tests/test_graph_scale_gpu.py tests/test_reference_suites_gpu.py tests/test_reference_swap_gpu.py tests/test_sharded_graph_gpu.py tests/test_spec_grids_gpu.py -q -p no:cacheprovider >> gpurun_out/jit2.txt 2>&1
cat gpurun_out/jit2.txt | tail -12
