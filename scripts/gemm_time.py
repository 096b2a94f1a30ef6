"""Kernel time of ops.gemm (bf16, bias + tanh-GELU, bf16 out) for square
sizes, CUDA events, median of 30; env AFG_GEMM_PAIR toggles CTA pairs."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import Epilogue, ops  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [2048, 4096, 8192]:
    a = (torch.rand(n, n, device="cuda") - 0.5).bfloat16()
    b = (torch.rand(n, n, device="cuda") - 0.5).bfloat16()
    bias = torch.rand(n, device="cuda")
    c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH, out=c)
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH, out=c)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"gemm {n}^3: {ms * 1e3:.1f} us  {2 * n**3 / ms / 1e9:.1f} TFLOP/s (min {ts[0]*1e3:.1f} us)",
          flush=True)
