"""Run by test_chains_gpu.test_stream_row_pool in a subprocess with
AFG_STREAM_POOL set (the library reads it once): the streamed softmax /
layernorm kernels with part of the rows claimed from the dynamic tail pool,
with and without a residual, checked against the oracle on sampled rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2603_06731_b200 import ops  # noqa: E402
from tests.gpu_util import check, to_host  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(9)
for rows, cols in ((32768, 768), (9001, 768), (5003, 1024)):
    x = (torch.rand((rows, cols), generator=g, device="cuda") * 2 - 1).bfloat16()
    r = (torch.rand((rows, cols), generator=g, device="cuda") * 2 - 1).bfloat16()
    gam = torch.rand(cols, generator=g, device="cuda") * 0.2 + 0.9
    bet = torch.rand(cols, generator=g, device="cuda") * 0.2 - 0.1
    idx = torch.arange(0, rows, 97, device="cuda")
    zero = torch.zeros((len(idx), cols), device="cuda").bfloat16()
    for res in (r, None):
        rr = r[idx] if res is not None else zero
        want = O.round_to(O.layernorm(to_host(x[idx]), to_host(rr), to_host(gam), to_host(bet),
                                      1e-12)[0], O.BF16)
        for _ in range(3):
            y = ops.layernorm_residual(x, res, gam, bet, eps=1e-12)
            check(to_host(y[idx]), want, 2.0**-7, f"layernorm {rows}x{cols} res={res is not None}")
for rows, cols in ((262144, 2048), (5003, 2048), (6000, 512)):
    x = (torch.rand((rows, cols), generator=g, device="cuda") * 8 - 4).half()
    idx = torch.arange(0, rows, 4099 if rows > 100000 else 97, device="cuda")
    want = O.round_to(O.softmax(to_host(x[idx])), O.F16)
    for _ in range(3):
        y = ops.softmax(x)
        check(to_host(y[idx]), want, 2.0**-10, f"softmax {rows}x{cols}")
torch.cuda.synchronize()
print("pool ok", os.environ.get("AFG_STREAM_POOL"))
