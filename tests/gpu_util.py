"""Helpers shared by the gpu tests: seeded inputs on the storage grid of a
dtype (generated with the reference generator so the oracle sees the very same
values), host<->device moves, and the reference's comparison rule."""
import numpy as np
import torch

import oracle as O

T_CODE = {torch.float32: O.F32, torch.float16: O.F16, torch.bfloat16: O.BF16}


def seeded(shape, name, seed, lo=-1.0, hi=1.0, dtype=torch.bfloat16):
    """makeRandomTensor values for buffer '%name' (interp.cpp:817-844), rounded
    (RNE) to `dtype`; returns (device tensor, float64 host copy of the exact
    stored values)."""
    host = O.round_to(O.random_tensor(tuple(shape), "%" + name, seed, lo, hi), T_CODE[dtype])
    dev = torch.from_numpy(host).to(dtype).to("cuda")
    # the device holds exactly `host` (both RNE from the same doubles)
    return dev, host


def to_host(t):
    return t.detach().float().cpu().double().numpy()


def check(got, want, tol, what=""):
    ok, ma, mr, w = O.compare(got, want, tol)
    assert ok, f"{what}: max_abs={ma:.3e} max_rel={mr:.3e} at {w} (tol {tol})"
    return mr
