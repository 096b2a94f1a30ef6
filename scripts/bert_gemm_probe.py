"""BERT-layer GEMM shapes (T = 64 x 512 tokens): time per epilogue variant
(graph-replayed, back to back, operands > L2 for the big ones)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06731_b200 import Epilogue, ops  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


T = 64 * 512
dev = "cuda"
for (K, N, name) in ((768, 2304, "qkv"), (768, 768, "out"), (768, 3072, "ffn1"), (3072, 768, "ffn2")):
    a = (torch.rand(T, K, device=dev) - 0.5).bfloat16()
    b = ((torch.rand(K, N, device=dev) - 0.5) * 0.05).bfloat16()
    bias = torch.rand(N, device=dev)
    res = (torch.rand(T, N, device=dev) - 0.5).bfloat16()
    c = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
    fl = 2.0 * T * N * K
    row = []
    for epi in (Epilogue.NONE, Epilogue.BIAS, Epilogue.BIAS_GELU_ERF, Epilogue.BIAS_GELU_TANH):
        us = timeit(lambda: ops.gemm(a, b, bias=bias, epilogue=epi, out=c))
        row.append(f"{epi.name} {us:6.1f}")
    us = timeit(lambda: ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS, residual=res, out=c))
    row.append(f"BIAS+res {us:6.1f}")
    us = timeit(lambda: torch.matmul(a, b, out=c))
    row.append(f"cublas {us:6.1f}")
    print(f"{name:5s} K={K} N={N}: " + "  ".join(row) + f"   (floor {fl / 1614e6:.1f} us)", flush=True)
