"""One GEMM shape (M K N epi), timed back to back under a CUDA graph; for
ncu captures of a single configuration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06731_b200 import Epilogue, Layout, ops  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
epi = Epilogue[sys.argv[4]] if len(sys.argv) > 4 else Epilogue.BIAS_RELU
a = (torch.rand(M, K, device="cuda") - 0.5).bfloat16()
b = ((torch.rand(N, K, device="cuda") - 0.5) * 0.1).bfloat16()
bias = torch.rand(N, device="cuda")
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
f = lambda: ops.gemm(a, b, bias=bias, epilogue=epi, b_layout=Layout.B_NK, out=c)  # noqa: E731
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
by = 2 * (M * K + N * K + M * N)
print(f"M={M} K={K} N={N} {epi.name}: {us:.1f} us, {by / us / 1e3:.0f} GB/s, {2 * M * N * K / us / 1e6:.0f} TFLOP/s")
