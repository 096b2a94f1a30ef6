"""CPU tests of the host-side graph API mirror (csrc/graph.cpp through the C
ABI afg_graph_check_json): the reference's parseGraphJson / checkGraph error
behaviour (test_frontend.cpp:253-273) and acceptance of every graph of the
reference's own tests and of the BASELINE patterns."""
import json
import os

import pytest

import paper_2603_06731_b200 as afg
from paper_2603_06731_b200.graph import check_graph

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "reference_graphs.json")))["cases"]


def test_parse_error_is_graph_error():
    with pytest.raises(afg.AfgError) as e:
        check_graph("{")
    assert e.value.status == 1 and "GraphError" in str(e.value)


def test_unsupported_op():
    g = {"tensors": [{"id": "a", "shape": [2]}, {"id": "b", "shape": [2]}],
         "ops": [{"op": "fancy", "inputs": ["a"], "output": "b"}]}
    with pytest.raises(afg.AfgError, match="unsupported-op"):
        check_graph(g)


def test_shape_mismatch():
    g = {"tensors": [{"id": "a", "shape": [2, 3]}, {"id": "b", "shape": [3, 4]},
                     {"id": "c", "shape": [2, 5]}],
         "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}
    with pytest.raises(afg.AfgError, match="shape-mismatch"):
        check_graph(g)


def test_missing_keys_and_unknown_dtype():
    with pytest.raises(afg.AfgError, match="tensors"):
        check_graph({"ops": []})
    with pytest.raises(afg.AfgError, match="dtype"):
        check_graph({"tensors": [{"id": "a", "shape": [1], "dtype": "f64"}], "ops": []})


def test_use_before_produce_and_duplicates():
    g = {"tensors": [{"id": "a", "shape": [2]}, {"id": "b", "shape": [2]}, {"id": "c", "shape": [2]}],
         "ops": [{"op": "add", "inputs": ["a", "c"], "output": "b"},
                 {"op": "exp", "inputs": ["b"], "output": "c"}]}
    with pytest.raises(afg.AfgError, match="used before"):
        check_graph(g)
    with pytest.raises(afg.AfgError, match="duplicate"):
        check_graph({"tensors": [{"id": "a", "shape": [1]}, {"id": "a", "shape": [1]}], "ops": []})


@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_reference_graphs_accepted(case):
    check_graph(case["graph"])
