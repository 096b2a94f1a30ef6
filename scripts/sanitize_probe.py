"""Small invocations of every mbarrier / TMA pipeline (K1 GEMM incl. a CTA-pair
and a stream-K shape, K2 conv im2col + halo, K3 attention, K4/K5 streamed
chains, K1c int8, the nest VM) for compute-sanitizer racecheck / synccheck /
memcheck runs (scripts/gpu_sanitize.sh)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_06731_b200 import Epilogue, ops  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
bf = torch.bfloat16
a = torch.randn(256, 512, device=dev).to(bf)
b = torch.randn(512, 512, device=dev).to(bf)
bias = torch.randn(512, device=dev)
ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH)                    # K1
ops.gemm(torch.randn(1024, 1024, device=dev).to(bf), torch.randn(1024, 1024, device=dev).to(bf),
         out_dtype=torch.float32)                                             # K1 (stream-K / pair)
x = torch.randn(1, 24, 24, 64, device=dev).to(bf)
w = torch.randn(64, 3, 3, 64, device=dev).to(bf) * 0.1
ops.conv2d_nhwc(x, w, torch.randn(64, device=dev), (1, 1), (1, 1), epilogue=Epilogue.BIAS_RELU)  # halo
ops.conv2d_nhwc(x, w, torch.randn(64, device=dev), (2, 2), (1, 1), epilogue=Epilogue.BIAS_RELU)  # im2col
q, k, v = (torch.randn(1, 2, 256, 128, device=dev).half() for _ in range(3))
ops.attention(q, k, v, scale=128 ** -0.5, causal=True)                          # K3
q2, k2, v2 = (torch.randn(1, 8, 1024, 64, device=dev).to(bf) for _ in range(3))
ops.attention(q2, k2, v2, scale=64 ** -0.5)                                    # K3, D=64, unit queue
xs = torch.randn(2048, 768, device=dev).to(bf)
ops.layernorm_residual(xs, xs, torch.ones(768, device=dev), torch.zeros(768, device=dev))  # K5
ops.layernorm_residual(xs, None, torch.ones(768, device=dev), torch.zeros(768, device=dev))  # no residual
ops.softmax(torch.randn(2048, 2048, device=dev).half())                         # K4
qa = torch.randint(-128, 128, (256, 256), dtype=torch.int8, device=dev)
ops.gemm_i8(qa, qa, out_mode=1, scale=1 / 1024)                                 # K1c
torch.cuda.synchronize()
print("sanitize probe done", flush=True)
