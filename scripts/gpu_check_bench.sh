#!/bin/bash
# GPU parity for the GEMM / conv / graph paths + the default bench line
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_graph_gpu.py tests/test_encoder_gpu.py tests/test_spec_grids_gpu.py tests/test_splitk_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1
tail -2 gpurun_out/pytest_part.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python scripts/summarize_bench.py gpurun_out/bench.json 2>&1 | tail -30
