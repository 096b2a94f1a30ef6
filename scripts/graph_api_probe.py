"""Host-clock phases of the graph API path (afg_graph_run, host doubles in /
out) on the BASELINE GEMM + GELU-composite graph at n^3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from oracle.graphs import matmul_epi_graph  # noqa: E402
from paper_2603_06731_b200.graph import execute  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g, fixed = matmul_epi_graph(n, n, n, "gelu")
t = time.perf_counter()
ins = O.random_graph_inputs(g, 7, -1.0, 1.0)
for k, v in fixed.items():
    ins[k] = v
for k in ("a", "b"):
    ins[k] = O.round_to(ins[k], O.BF16)
print(f"inputs {time.perf_counter() - t:.2f} s", flush=True)
text = json.dumps(g)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t = time.perf_counter()
    out = execute(text, ins)
    print(f"execute {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
