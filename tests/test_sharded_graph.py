"""Host side of the thread-per-device sharded graph execution
(GpuOptions::devices, afg_graph_run_sharded): the dim-0 shard propagation
accepts batch-separable graphs and rejects graphs that mix rows across shards
with a GraphError -- checked on CPU (a shardable graph then fails only for
want of a device: InterpError, status 3)."""
import json
import os

import pytest

import paper_2603_06731_b200 as afg
from paper_2603_06731_b200.graph import execute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _case(name):
    spec = json.load(open(os.path.join(GOLD, "scale_graphs.json")))["cases"]
    return next(c for c in spec if c["name"] == name)


def _zeros(graph):
    import numpy as np
    produced = {o["output"] for o in graph["ops"]}
    return {t["id"]: np.zeros(t["shape"]) for t in graph["tensors"] if t["id"] not in produced}


def test_bert_graph_not_shardable_along_rows():
    g = _case("bert_layer_graph_s64_h128")["graph"]
    with pytest.raises(afg.AfgError, match="not shardable") as e:
        execute(g, _zeros(g), devices=[0, 0])
    assert e.value.status == 1


@pytest.mark.parametrize("name", ["gemm_bf16_relu_512x256x384", "nhwc_conv3x3_same_16x16_64to128"])
def test_batch_separable_graphs_pass_the_shard_plan(name):
    if afg.lib().afg_device_count() > 0:
        pytest.skip("CPU-side check (a GPU runs the shards: tests/test_sharded_graph_gpu.py)")
    g = _case(name)["graph"]
    with pytest.raises(afg.AfgError) as e:
        execute(g, _zeros(g), devices=[0, 0])
    assert e.value.status == 3, str(e.value)  # no device -- not a GraphError
