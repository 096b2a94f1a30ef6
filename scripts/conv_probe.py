"""Device time of single NHWC conv layers (bf16, bias + ReLU), CUDA-graph
replay behind a GPU spin, median of 20. Args: B,H,C,OC,k,s ..."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import Epilogue, ops  # noqa: E402

for spec in sys.argv[1:]:
    B, H, C, OC, k, s = (int(v) for v in spec.split(","))
    p = 1 if k == 3 else 0
    x = (torch.rand(B, H, H, C, device="cuda") - 0.5).bfloat16()
    w = (torch.rand(OC, k, k, C, device="cuda") - 0.5).bfloat16() * 0.1
    b = torch.rand(OC, device="cuda")
    fn = lambda: ops.conv2d_nhwc(x, w, b, (s, s), (p, p), epilogue=Epilogue.BIAS_RELU)  # noqa: E731
    fn()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    for e0, e1 in evs:
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) for e0, e1 in evs)[10]
    OH = (H + 2 * p - k) // s + 1
    fl = 2.0 * B * OH * OH * OC * C * k * k
    print(f"conv B{B} {H}x{H}x{C}->{OC} k{k} s{s}: {t*1e3:.1f} us {fl/t/1e9:.0f} TFLOP/s", flush=True)
