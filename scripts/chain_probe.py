"""Device time of the layernorm / softmax chains vs row count (CUDA graph
replay behind a GPU spin, L2 flushed by a 256 MB write + read before each)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import ops  # noqa: E402

flw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flr = torch.zeros(64 << 20, device="cuda")


def timeit(fn, n=10):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    fn()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    for a, b in evs:
        flw.zero_()
        flr.sum()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    return t[len(t) // 2]


for rows in (8192, 32768, 131072):
    cols = 768
    x = torch.rand(rows, cols, device="cuda").bfloat16()
    r = torch.rand(rows, cols, device="cuda").bfloat16()
    gm = torch.rand(cols, device="cuda")
    bt = torch.rand(cols, device="cuda")
    y = torch.empty_like(x)
    ms = timeit(lambda: ops.layernorm_residual(x, r, gm, bt, out=y))
    print(f"layernorm [{rows},{cols}] {ms*1e3:.1f} us {3*rows*cols*2/ms/1e6:.0f} GB/s", flush=True)
for rows in (32768, 262144):
    x = torch.rand(rows, 2048, device="cuda").half()
    y = torch.empty_like(x)
    ms = timeit(lambda: ops.softmax(x, out=y))
    print(f"softmax [{rows},2048] {ms*1e3:.1f} us {2*rows*2048*2/ms/1e6:.0f} GB/s", flush=True)
x = torch.rand(1 << 28, device="cuda").bfloat16()
y = torch.empty_like(x)
ms = timeit(lambda: y.copy_(x))
print(f"torch copy 512MB {ms*1e3:.1f} us {2*x.numel()*2/ms/1e6:.0f} GB/s", flush=True)
x = torch.rand(3 * 32768 * 768 // 2, device="cuda").bfloat16()
y = torch.empty_like(x)
ms = timeit(lambda: y.copy_(x))
print(f"torch copy {x.numel()*2/1e6:.0f} MB {ms*1e3:.1f} us {2*x.numel()*2/ms/1e6:.0f} GB/s", flush=True)
