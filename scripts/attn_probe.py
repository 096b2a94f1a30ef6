"""Runs one attention config in this process (for per-config isolation
under `timeout`): prints PASS/FAIL and the max error vs the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2603_06731_b200 import ops  # noqa: E402
from tests.gpu_util import seeded, to_host  # noqa: E402

B, H, N, D, causal = (int(v) for v in sys.argv[1:6])
dt = torch.float16
q, qh = seeded((B, H, N, D), "q", 36, dtype=dt)
k, kh = seeded((B, H, N, D), "k", 36, dtype=dt)
v, vh = seeded((B, H, N, D), "v", 36, dtype=dt)
o = ops.attention(q, k, v, causal=bool(causal), out_dtype=torch.float32)
torch.cuda.synchronize()
got = to_host(o)
want = O.attention(qh, kh, vh, causal=bool(causal))
ok, ma, mr, w = O.compare(got, want, 2e-3)
print(("PASS" if ok else "FAIL"), sys.argv[1:6], f"max_rel={mr:.3e} worst={w}", flush=True)
