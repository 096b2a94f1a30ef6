"""Kernel time of ops.gemm_i8 (i8 x i8 -> i32 / requantised i8) for square
sizes: CUDA events, median of 20, L2 flushed between launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import ops  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in [int(x) for x in sys.argv[1:]] or [4096, 8192]:
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    for mode in (0, 1):
        c = ops.gemm_i8(a, b, out_mode=mode, scale=1e-4)
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.gemm_i8(a, b, out_mode=mode, scale=1e-4, out=c)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        print(f"i8 gemm {n}^3 mode {mode}: {ms*1e3:.1f} us  {2*n**3/ms/1e9:.1f} TOP/s", flush=True)
