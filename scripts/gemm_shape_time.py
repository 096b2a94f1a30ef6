"""Kernel time of ops.gemm (bf16 in / bf16 out) for M,N,K,epilogue shapes given
as "MxNxK:epi[:kn]" arguments (epi = none|relu|gelu|erf), CUDA events, median of 30
with an L2 flush between launches. Env knobs (AFG_GEMM_*) select variants."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import Epilogue, Layout, ops  # noqa: E402

EPI = {"none": Epilogue.NONE, "relu": Epilogue.BIAS_RELU, "gelu": Epilogue.BIAS_GELU_TANH,
       "erf": Epilogue.BIAS_GELU_ERF, "bias": Epilogue.BIAS}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for spec in sys.argv[1:]:
    shape, epi, *lay = spec.split(":")
    kn = lay == ["kn"]
    m, n, k = (int(x) for x in shape.split("x"))
    a = (torch.rand(m, k, device="cuda") - 0.5).bfloat16()
    b = (torch.rand(*((k, n) if kn else (n, k)), device="cuda") - 0.5).bfloat16()
    bias = torch.rand(n, device="cuda")
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    kw = {} if epi == "none" else {"bias": bias}
    for _ in range(3):
        ops.gemm(a, b, epilogue=EPI[epi], out=c, b_layout=Layout.B_KN if kn else Layout.B_NK, **kw)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.gemm(a, b, epilogue=EPI[epi], out=c, b_layout=Layout.B_KN if kn else Layout.B_NK, **kw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{spec}: {ms * 1e3:.1f} us  {2 * m * n * k / ms / 1e9:.1f} TFLOP/s (min {ts[0]*1e3:.1f})",
          flush=True)
