"""One NHWC conv (B H C OC k stride), timed back to back (bf16, bias+ReLU)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06731_b200 import Epilogue, check, lib  # noqa: E402

B, H, C, OC, k, s = (int(v) for v in sys.argv[1:7])
pad = 1 if k == 3 else 0
OH = (H + 2 * pad - k) // s + 1
x = (torch.rand(B, H, H, C, device="cuda") - 0.5).bfloat16()
w = ((torch.rand(OC, k, k, C, device="cuda") - 0.5) * 0.1).bfloat16()
bias = torch.rand(OC, device="cuda")
y = torch.empty(B, OH, OH, OC, device="cuda", dtype=torch.bfloat16)
L = lib()
f = lambda: check(L.afg_conv2d_nhwc(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), B, H, H, C, OC,  # noqa
                                    k, k, s, s, pad, pad, 1, 1, OH, OH, 2, int(Epilogue.BIAS_RELU),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
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
fl = 2.0 * B * OH * OH * OC * C * k * k
print(f"B{B} {H} {C}->{OC} k{k} s{s}: {us:.1f} us {fl / us / 1e6:.0f} TFLOP/s "
      f"[BN={os.environ.get('AFG_CONV_BN', 'auto')} pair={os.environ.get('AFG_GEMM_PAIR', '1')}]")
