"""Times the fused attention kernel alone (CUDA events, median of 20) for the
BASELINE shape; used with AFG_ATTN_DEBUG to split softmax vs MMA cost."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import ops  # noqa: E402

B, H, N, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 16, 2048, 128)
torch.manual_seed(0)
q, k, v = (torch.rand(B, H, N, D, device="cuda").half() * 2 - 1 for _ in range(3))
for causal in (0, 1):
    o = torch.empty_like(q)
    for _ in range(3):
        ops.attention(q, k, v, scale=D ** -0.5, causal=bool(causal), out=o)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.attention(q, k, v, scale=D ** -0.5, causal=bool(causal), out=o)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    fl = 4 * B * H * N * N * D * (0.5 if causal else 1.0)
    print(f"B{B} H{H} N{N} D{D} dbg={os.environ.get('AFG_ATTN_DEBUG', '0')} causal={causal} {ms*1e3:.1f} us "
          f"{fl / ms / 1e9:.1f} TFLOP/s", flush=True)
