#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
{
for sk in 1 0; do for n in 2048 4096; do AFG_GEMM_STREAMK=$sk python bench.py --workload gemm_bf16 --size $n --only --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sk=$sk n=$n', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done; done
for w in layernorm bert_layer; do timeout 300 python bench.py --workload $w --only --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
} > gpurun_out/perf4.txt 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_chains_gpu.py tests/test_encoder_gpu.py tests/test_splitk_gpu.py tests/test_graph_scale_gpu.py -q -p no:cacheprovider >> gpurun_out/perf4.txt 2>&1
python - >> gpurun_out/perf4.txt 2>&1 <<'PY'
# stream-K parity at 2048^3 (and ragged) vs the oracle on sampled rows
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle as O
from paper_2603_06731_b200 import ops, Epilogue
from tests.gpu_util import seeded, to_host
for (M, N, K) in [(2048, 2048, 2048), (1920, 2304, 1536), (2048, 1024, 4096)]:
    a, ah = seeded((M, K), "a", 3); b, bh = seeded((K, N), "b", 3)
    bias, biash = seeded((N,), "bias", 3, dtype=torch.float32)
    for _ in range(3):
        c = ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH, out_dtype=torch.float32)
    rows = np.arange(0, M, 61)
    want = O.matmul(ah[rows], bh, biash, epi=O.EPI_GELU_TANH, out_t=O.F64)
    ok, ma, mr, w = O.compare(to_host(c)[rows], want, 1e-5)
    print("streamk parity", M, N, K, ok, mr)
PY
tail -40 gpurun_out/perf4.txt
