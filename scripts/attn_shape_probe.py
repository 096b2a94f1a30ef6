"""Attention at one shape (B H N D dtype causal), timed back to back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06731_b200 import ops  # noqa: E402

B, H, N, D = (int(v) for v in sys.argv[1:5])
dt = torch.bfloat16 if (len(sys.argv) > 5 and sys.argv[5] == "bf16") else torch.float16
causal = len(sys.argv) > 6 and sys.argv[6] == "1"
q, k, v = ((torch.rand(B, H, N, D, device="cuda") - 0.5).to(dt) for _ in range(3))
f = lambda: ops.attention(q, k, v, scale=D ** -0.5, causal=causal)  # noqa: E731
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
fl = 4.0 * B * H * N * N * D * (0.5 if causal else 1.0)
print(f"B{B} H{H} N{N} D{D} {dt} causal={causal} dbg={os.environ.get('AFG_ATTN_DEBUG', '0')}: "
      f"{us:.1f} us {fl / us / 1e6:.0f} TFLOP/s")
