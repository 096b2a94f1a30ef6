"""2048^3 / 4096^3 GEMM probe: the bench measurement (L2 flushed, graph
replay, mean) with different epilogues; env knobs are passed by the caller."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_06731_b200 import Epilogue  # noqa: E402

ctx = bench.Ctx(0, 1, 0)
for n in [int(a) for a in sys.argv[1:]] or [2048]:
    for epi in (Epilogue.NONE, Epilogue.BIAS, Epilogue.BIAS_GELU_TANH):
        wl = bench.GemmBF16(n)
        wl.step = (lambda w, e: lambda: w.ops.gemm(w.A, w.B, bias=w.bias, epilogue=e, out=w.C))(wl, epi)
        m = bench.measure(ctx, wl, 50, 5)
        print(f"n={n} epi={epi.name:16s} {m['value']:8.1f} TFLOP/s  {m['ms_per_step'] * 1e3:7.2f} us "
              f"env={os.environ.get('PROBE_TAG', '')}", flush=True)
        bench.release(wl)
