"""Runs one large fused VM region (the 14-nest GELU composite on a
[2048, 4096] f32 tensor, one launch) through the graph executor; used for the
nest-VM ncu capture and timing (prints device ms of the executor call)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle.graphs import matmul_epi_graph  # noqa: E402
from paper_2603_06731_b200.graph import execute  # noqa: E402

M, N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g, fixed = matmul_epi_graph(M, N, 8, "gelu")
g["ops"] = [o for o in g["ops"] if o["output"] not in ("c", "bb", "cb")]
g["tensors"] = [t for t in g["tensors"] if t["id"] not in ("a", "b", "bias", "c", "bb")]
rng = np.random.default_rng(0)
inputs = {"cb": rng.uniform(-3, 3, (M, N))}
inputs.update(fixed)
for i in range(3):
    t0 = time.perf_counter()
    out, plan = execute(g, inputs, want_plan=True)
    print(f"run {i}: {1e3 * (time.perf_counter() - t0):.1f} ms host wall; plan {plan}", flush=True)
