"""1x1-conv store path probe: afg conv vs cuBLAS matmul of the same GEMM vs a
pure write / copy of the output bytes (what the HBM actually gives)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06731_b200 import Epilogue, check, lib  # noqa: E402

L = lib()
dev = torch.device("cuda:0")


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


shapes = [(56, 64, 256), (56, 256, 64), (28, 128, 512), (14, 256, 1024), (14, 1024, 256), (7, 512, 2048)]
for H, C, OC in shapes:
    B = 256
    x = (torch.rand(B, H, H, C, device=dev) - 0.5).to(torch.bfloat16)
    w = (torch.rand(OC, 1, 1, C, device=dev) - 0.5).to(torch.bfloat16) * 0.1
    bias = torch.rand(OC, device=dev)
    y = torch.empty(B, H, H, OC, device=dev, dtype=torch.bfloat16)
    conv = lambda: check(L.afg_conv2d_nhwc(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), B, H, H, C, OC,  # noqa
                                           1, 1, 1, 1, 0, 0, 1, 1, H, H, 2, int(Epilogue.BIAS_RELU),
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    x2, w2, y2 = x.view(-1, C), w.view(OC, C).t(), y.view(-1, OC)
    mm = lambda: torch.matmul(x2, w2, out=y2)  # noqa
    wr = lambda: y.zero_()  # noqa
    big = torch.empty_like(y)
    cp = lambda: big.copy_(y)  # noqa
    by = 2 * (x.numel() + y.numel() + w.numel())
    r = {k: timeit(f) for k, f in (("afg", conv), ("cublas", mm), ("write_y", wr), ("copy_y", cp))}
    print(f"{H:3d} {C:5d}->{OC:5d}: " + "  ".join(f"{k} {v:7.1f} us" for k, v in r.items()) +
          f"   afg {by / r['afg'] / 1e3:6.0f} GB/s  write {2 * y.numel() / r['write_y'] / 1e3:6.0f} GB/s"
          f"  copy {4 * y.numel() / r['copy_y'] / 1e3:6.0f} GB/s", flush=True)
