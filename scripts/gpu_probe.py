"""Quick GPU probe: correctness of the first kernels vs torch fp32 and a timing
of the headline GEMM. Development aid (not a test, not the bench)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_06731_b200 as afg  # noqa: E402
from paper_2603_06731_b200 import ops, Epilogue, Layout  # noqa: E402


def rel_err(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).abs() / torch.clamp(torch.maximum(a.abs(), b.abs()), min=1.0)).max().item()


def check_gemm(M, N, K, dt=torch.bfloat16, epi=Epilogue.BIAS_GELU_TANH, layout=Layout.B_KN, od=None):
    torch.manual_seed(0)
    a = (torch.rand(M, K, device="cuda") * 2 - 1).to(dt)
    if layout == Layout.B_KN:
        b = (torch.rand(K, N, device="cuda") * 2 - 1).to(dt)
        bf = b.float()
    else:
        b = (torch.rand(N, K, device="cuda") * 2 - 1).to(dt)
        bf = b.float().t()
    bias = torch.rand(N, device="cuda") * 2 - 1
    c = ops.gemm(a, b, bias=bias, epilogue=epi, b_layout=layout, out_dtype=od)
    torch.cuda.synchronize()
    ref = a.float() @ bf + bias
    if epi == Epilogue.BIAS_GELU_TANH:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    elif epi == Epilogue.BIAS_RELU:
        ref = torch.relu(ref)
    elif epi == Epilogue.NONE:
        ref = a.float() @ bf
    e = rel_err(c, ref)
    print(f"gemm M={M} N={N} K={K} {dt} layout={int(layout)} epi={int(epi)} out={c.dtype}: maxrel={e:.3e}", flush=True)
    return e


def main():
    print("devices", afg.lib().afg_device_count(), torch.cuda.get_device_name(0), flush=True)
    errs = []
    for (M, N, K) in [(128, 256, 64), (256, 256, 128), (128, 128, 64), (100, 200, 72), (1024, 1024, 1024),
                      (512, 768, 768), (333, 130, 200)]:
        errs.append(check_gemm(M, N, K))
    errs.append(check_gemm(512, 512, 256, layout=Layout.B_NK))
    errs.append(check_gemm(512, 512, 256, dt=torch.float16, epi=Epilogue.BIAS_RELU, od=torch.float32))
    errs.append(check_gemm(256, 64, 128, epi=Epilogue.NONE))
    errs.append(check_gemm(64, 64, 64, dt=torch.float32, epi=Epilogue.BIAS_RELU))
    # softmax / layernorm
    x = torch.randn(1000, 2048, device="cuda", dtype=torch.float16)
    y = ops.softmax(x)
    print("softmax maxrel", rel_err(y, torch.softmax(x.float(), -1)), flush=True)
    xb = torch.randn(1000, 768, device="cuda", dtype=torch.bfloat16)
    rb = torch.randn(1000, 768, device="cuda", dtype=torch.bfloat16)
    g = torch.rand(768, device="cuda")
    be = torch.rand(768, device="cuda")
    yl = ops.layernorm_residual(xb, rb, g, be, eps=1e-12)
    ref = torch.nn.functional.layer_norm(xb.float() + rb.float(), (768,), g, be, eps=1e-12)
    print("layernorm maxrel", rel_err(yl, ref), flush=True)

    # timing 8192^3 bf16 GELU
    for n in (4096, 8192):
        a = (torch.rand(n, n, device="cuda") * 2 - 1).to(torch.bfloat16)
        b = (torch.rand(n, n, device="cuda") * 2 - 1).to(torch.bfloat16)
        bias = torch.rand(n, device="cuda")
        out = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 10
        s.record()
        for _ in range(it):
            ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH, out=out)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / it
        print(f"afg gemm {n}^3: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        s.record()
        for _ in range(it):
            torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / it
        print(f"torch matmul {n}^3: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
    print("MAXERR", max(errs))


if __name__ == "__main__":
    main()
