"""Binding of the C++ graph executor (csrc/graph.cpp, include/afg_graph.h):
the drop-in for the reference's parseGraphJson -> lowerGraphToAffine ->
af::interpret path. Inputs and outputs are host arrays of doubles, keyed like
the reference's interpreter ("%id")."""
from __future__ import annotations

import ctypes
import json

import numpy as np

from . import AfgError, lib


def check_graph(graph) -> None:
    """Graph JSON read + table-driven validation with checkGraph's error
    behaviour (GraphError -> AfgError status 1)."""
    text = graph if isinstance(graph, str) else json.dumps(graph)
    L = lib()
    st = L.afg_graph_check_json(text.encode())
    if st != 0:
        raise AfgError(st, L.afg_last_error().decode(errors="replace"))


FUSE = 1
EXACT = 2


def execute(graph, inputs: dict, fuse: bool = True, stream=None, want_plan=False,
            exact: bool = False, devices=None, shard_extent: int = 0):
    """Runs the graph on the GPU. inputs: {id or %id: array}. Returns
    {"%id": float64 array} (and the executed kernel plan if want_plan).
    fuse: kernel patterns + fused VM regions (else one launch per op);
    exact: keep f32 tensors off the tensor cores (bit-exact paths only);
    devices: run sharded, one host thread per entry (the leading extent
    shard_extent, default the first input's, split into contiguous blocks)."""
    text = graph if isinstance(graph, str) else json.dumps(graph)
    L = lib()
    names = list(inputs)
    arrs = [np.ascontiguousarray(np.asarray(inputs[n], dtype=np.float64)).ravel() for n in names]
    DP = ctypes.POINTER(ctypes.c_double)
    c_names = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    c_data = (DP * len(names))(*[a.ctypes.data_as(DP) for a in arrs])
    c_numel = (ctypes.c_int64 * len(names))(*[a.size for a in arrs])
    out = ctypes.c_void_p()
    flags = (FUSE if fuse else 0) | (EXACT if exact else 0)
    if devices:
        devs = (ctypes.c_int * len(devices))(*devices)
        st = L.afg_graph_run_sharded(text.encode(), len(names), c_names, c_data, c_numel, flags,
                                     len(devices), devs, int(shard_extent), ctypes.byref(out))
    else:
        st = L.afg_graph_run(text.encode(), len(names), c_names, c_data, c_numel, flags,
                             stream, ctypes.byref(out))
    if st != 0:
        raise AfgError(st, L.afg_last_error().decode(errors="replace"))
    try:
        res = {}
        for i in range(L.afg_graph_result_count(out)):
            name = L.afg_graph_result_name(out, i).decode()
            shape = tuple(L.afg_graph_result_dim(out, i, d)
                          for d in range(L.afg_graph_result_rank(out, i)))
            n = L.afg_graph_result_numel(out, i)
            p = L.afg_graph_result_data(out, i)
            res[name] = np.ctypeslib.as_array(p, shape=(n,)).copy().reshape(shape)
        plan = L.afg_graph_result_plan(out).decode()
    finally:
        L.afg_graph_result_free(out)
    return (res, plan.splitlines()) if want_plan else res
