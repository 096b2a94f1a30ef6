import sys
import torch
sys.path.insert(0, ".")
from paper_2603_06731_b200 import ops
for rows in [int(v) for v in sys.argv[1:]]:
    x = torch.rand(rows, 768, device="cuda").bfloat16()
    r = torch.rand(rows, 768, device="cuda").bfloat16()
    g = torch.rand(768, device="cuda")
    b = torch.rand(768, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        ops.layernorm_residual(x, r, g, b, out=y)
    torch.cuda.synchronize()
