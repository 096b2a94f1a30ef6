"""Kernel time of one ops.gemm call for a given M N K / epilogue (CUDA events,
median of 30)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import Epilogue, ops  # noqa: E402


def run(M, N, K, epi, out_dt=torch.bfloat16):
    a = (torch.rand(M, K, device="cuda") - 0.5).bfloat16()
    b = (torch.rand(K, N, device="cuda") - 0.5).bfloat16()
    bias = torch.rand(N, device="cuda")
    c = torch.empty(M, N, device="cuda", dtype=out_dt)
    for _ in range(3):
        ops.gemm(a, b, bias=bias, epilogue=epi, out=c)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            ops.gemm(a, b, bias=bias, epilogue=epi, out=c)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(30)]
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)  # the host enqueues every replay while the GPU spins
    for e0, e1 in evs:
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) for e0, e1 in evs]
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"gemm {M}x{N}x{K} epi={int(epi)} out={out_dt}: {ms * 1e3:.1f} us "
          f"{2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)


for spec in sys.argv[1:]:
    M, N, K, e = (int(x) for x in spec.split(","))
    run(M, N, K, Epilogue(e))
