"""Kernel time of ops.conv2d_nhwc_i8 on ResNet-50-like layers (batch 256):
CUDA events, median of 10, L2 flushed between launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import ops  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (H, C, OC, K, s) in [(56, 64, 64, 3, 1), (28, 128, 128, 3, 1), (14, 256, 256, 3, 1),
                         (56, 64, 256, 1, 1), (14, 256, 1024, 1, 1)]:
    B = 256
    x = torch.randint(-128, 128, (B, H, H, C), dtype=torch.int8, device="cuda")
    w = torch.randint(-128, 128, (OC, K, K, C), dtype=torch.int8, device="cuda")
    p = K // 2
    ops.conv2d_nhwc_i8(x, w, stride=(s, s), pad=(p, p), out_mode=1, scale=1e-4)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.conv2d_nhwc_i8(x, w, stride=(s, s), pad=(p, p), out_mode=1, scale=1e-4)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    OH = (H + 2 * p - K) // s + 1
    ops_ = 2.0 * B * OH * OH * OC * K * K * C
    print(f"i8 conv {H}x{H} {C}->{OC} k{K} s{s}: {ms*1e3:.1f} us  {ops_/ms/1e9:.1f} TOP/s", flush=True)
