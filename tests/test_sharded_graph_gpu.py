"""Thread-per-device sharded graph execution on the B200 (GpuOptions::devices
= [0, 0]: two shards, two host threads, sharing the one GPU): the leading
(row / batch) dimension is split, each shard runs the full planner (tensor-
core patterns included), the outputs are concatenated -- and must equal both
the unsharded run (bit-identical: every row is computed by the same kernel
arithmetic) and the reference interpreter's outputs (the scale goldens)."""
import numpy as np
import pytest

import oracle as O
from paper_2603_06731_b200.graph import execute
from tests.test_graph_scale_gpu import GOLD, SPEC, build_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["gemm_bf16_relu_512x256x384", "nhwc_conv3x3_same_16x16_64to128",
                                  "nhwc_conv3x3_s2_prepadded_34", "gelu_composite_region_64x96"])
def test_sharded_equals_unsharded_and_reference(cuda, name):
    case = next(c for c in SPEC if c["name"] == name)
    ins = build_inputs(case)
    whole = execute(case["graph"], ins)
    shard, plan = execute(case["graph"], ins, devices=[0, 0], want_plan=True)
    assert any("[shard 1" in p for p in plan), plan
    for k in case["outputs"]:
        assert np.array_equal(shard[k], whole[k]), k
        ok, ma, mr, w = O.compare(shard[k], GOLD[f"{name}/{k}"].astype(np.float64),
                                  case["tol"] if case["tol"] > 0 else 0.0)
        assert ok, f"{name} {k}: {mr}"
