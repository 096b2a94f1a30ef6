#!/usr/bin/env python3
"""bench.py - headline benchmark of the afg B200 kernels (BASELINE.json).

Default workload (BASELINE configs[1]): bf16 matmul 16384^3, fp32
accumulation, fused bias + tanh-GELU epilogue, row-sharded across ranks
(strong scaling: the 16384^3 problem is fixed, each rank computes M/N rows
against the full B). One step = one pass of the hot path (one fused GEMM
launch) over one batch of synthetic input already resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--impl afg|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL for barriers and the
max-over-ranks reduction of the device time; no data-path collective).
--impl reference times the reference's own CPU path (the AffineForge
interpreter, oracle/_ref, or the oracle C port if it is absent) on the
host cores with every thread, on a bounded sample of the same workload.

Prints ONE JSON line (rank 0). The default run (workload gemm_bf16, no
--only) also measures every other BASELINE config in the same process and
reports them under "workloads": the GEMM sweep sizes, fp32 1024^3, attention
(causal and not), the ResNet-50 conv set, the BERT layer, softmax, layernorm,
int8 GEMM and the split-K tensor-parallel GEMM -- each with its value, the
roofline fraction (same statistic as value: the mean step time), the clocks
and the ncu DRAM traffic of its dominant kernel.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained"), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback"}


def fp32_simt_peak(clk):
    """FP32 CUDA-core peak of the B200: 148 SMs x 128 FP32 lanes x 2 flop per
    FMA x the SM clock (the max clock nvidia-smi reports, else 1965 MHz)."""
    mhz = (clk or {}).get("sm_max_mhz") or 1965.0
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def floor_fields(wl, peaks, k_ms):
    """Multi-kernel steps mixing tensor- and HBM-bound ops (ResNet convs, the
    BERT layer): the sum over ops of max(flops / tensor peak, bytes / HBM peak)
    and the step's fraction of it, next to the tensor-only `frac`."""
    ops = getattr(wl, "ops_fb", None)
    if not ops:
        return {}
    floor_s = sum(c * max(f / (peaks["bf16_tflops"] * 1e12), b / (peaks["hbm_gbs"] * 1e9))
                  for c, f, b in ops)
    return {"op_floor_ms": floor_s * 1e3, "frac_of_op_floor": floor_s * 1e3 / k_ms}


def traffic_for(workload):
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# ------------------------------------------------------------- clocks ---

class L2Flush:
    """Untimed L2 flush between steps: write a 256 MB buffer (> the 126 MB L2),
    then read a second 256 MB buffer so the L2 ends up holding clean lines --
    the timed step then pays neither cached operands nor the flush's own dirty
    write-backs."""

    def __init__(self, dev):
        import torch
        self.w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def __call__(self):
        self.w.zero_()
        self.r.sum()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    self.samples.append(parts)

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in self.samples:
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------- distributed ---

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


from paper_2603_06731_b200.shard import shard_rows, shard_seed  # noqa: E402


# ============================================================ workloads ===

class GemmBF16:
    """BASELINE configs[1]: bf16 C = gelu_tanh(A B + bias), fp32 accumulate."""

    def __init__(self, size):
        self.n = size
        self.name = f"gemm_bf16_gelu_{size}"  # per-size traffic entry in profiles/traffic.json
        # A, B and C fit in the 126 MB L2 up to 4096^2: flush between steps
        self.flushed = 3 * 2 * size * size < 2 * 126e6 and not os.environ.get("AFG_BENCH_NO_FLUSH")
        self.flush = None

    def config(self, world):
        return {"workload": f"bf16 matmul {self.n}x{self.n}x{self.n} + bias + tanh-GELU "
                            f"epilogue (fp32 accumulate), row-sharded",
                "M": self.n, "N": self.n, "K": self.n, "parallelism": f"rows/{world}",
                "l2": ("operands larger than L2 (no flush needed)" if not self.flushed else
                       "L2 flushed between steps (256 MB write + 256 MB read, untimed)"),
                "sweep": "2048-16384 via --size"}

    metric = "TFLOP/s"
    unit = "TFLOP/s"
    dtype = "bf16"
    bound = "tensor"

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import ops
        self.torch = torch
        self.ops = ops
        r0, r1 = shard_rows(self.n, rank, world)
        self.m = r1 - r0
        import oracle  # generator seed only: the data are made on the device
        self.A = ops.fill_uniform((self.m, self.n), shard_seed(oracle.stream_seed("%a", 1),
                                                               r0 * self.n), -1, 1, torch.bfloat16)
        self.B = ops.fill_uniform((self.n, self.n), oracle.stream_seed("%b", 1), -1, 1,
                                  torch.bfloat16)
        self.bias = ops.fill_uniform((self.n,), oracle.stream_seed("%bias", 1), -1, 1,
                                     torch.float32)
        self.C = torch.empty((self.m, self.n), dtype=torch.bfloat16, device=dev)
        if self.flushed:
            self.flush = L2Flush(dev)
            self.pre_step = self.flush
        self.flops_rank = 2.0 * self.m * self.n * self.n
        self.flops_total = 2.0 * self.n ** 3
        self.alg_bytes_rank = 2.0 * (self.m * self.n + self.n * self.n + self.m * self.n) + 4 * self.n

    def step(self):
        from paper_2603_06731_b200 import Epilogue
        self.ops.gemm(self.A, self.B, bias=self.bias, epilogue=Epilogue.BIAS_GELU_TANH, out=self.C)

    def launches_per_step(self):
        return 1

    # e2e: pinned host bf16 buffers -> H2D -> afg_gemm (C ABI) -> D2H, the rows
    # of A / C pipelined in chunks over the two copy engines: chunk i's GEMM
    # overlaps chunk i+1's H2D and chunk i-1's D2H
    e2e_path = ("pinned host -> H2D (copy stream) -> afg_gemm per 1/8 of the rows -> D2H (second "
                "copy stream), chunks overlapped; B and bias copied once per step")

    def e2e_setup(self):
        t = self.torch
        self.hA = self.A.cpu().pin_memory()
        self.hB = self.B.cpu().pin_memory()
        self.hbias = self.bias.cpu().pin_memory()
        self.hC = t.empty((self.m, self.n), dtype=t.bfloat16).pin_memory()
        self.dA = t.empty_like(self.A)
        self.dB = t.empty_like(self.B)
        self.dbias = t.empty_like(self.bias)
        self.h2d = self.hA.numel() * 2 + self.hB.numel() * 2 + self.hbias.numel() * 4
        self.d2h = self.hC.numel() * 2
        self.s_in, self.s_out = t.cuda.Stream(), t.cuda.Stream()
        step = max(256, -(-self.m // 8) // 256 * 256)
        self.chunks = [(r, min(self.m, r + step)) for r in range(0, self.m, step)]

    def e2e_step(self):
        from paper_2603_06731_b200 import Epilogue
        t = self.torch
        cur = t.cuda.current_stream()
        self.s_in.wait_stream(cur)
        ev_in, ev_out = [], []
        with t.cuda.stream(self.s_in):
            self.dB.copy_(self.hB, non_blocking=True)
            self.dbias.copy_(self.hbias, non_blocking=True)
            for r0, r1 in self.chunks:
                self.dA[r0:r1].copy_(self.hA[r0:r1], non_blocking=True)
                e = t.cuda.Event()
                e.record(self.s_in)
                ev_in.append(e)
        for (r0, r1), e in zip(self.chunks, ev_in):
            cur.wait_event(e)
            self.ops.gemm(self.dA[r0:r1], self.dB, bias=self.dbias,
                          epilogue=Epilogue.BIAS_GELU_TANH, out=self.C[r0:r1])
            o = t.cuda.Event()
            o.record(cur)
            ev_out.append(o)
        for (r0, r1), o in zip(self.chunks, ev_out):
            self.s_out.wait_event(o)
            with t.cuda.stream(self.s_out):
                self.hC[r0:r1].copy_(self.C[r0:r1], non_blocking=True)
        cur.wait_stream(self.s_out)

    # bounded CPU sample of the same workload through the reference path
    def reference_sample(self, threads):
        return ReferenceGemmSample(self.n, threads)


class GemmSplitK:
    """North-star item 4 / SURVEY §8e: the split-K tensor-parallel GEMM, the
    one config with an exchange step. bf16 16384^3 + bias + tanh-GELU; the K
    dimension is split across ranks, each computes its fp32 partial on the
    tensor cores, NCCL reduce-scatters the partials over NVLink into row
    blocks, the epilogue runs on the reduced rows (afg_gemm_splitk)."""

    metric = "TFLOP/s"
    unit = "TFLOP/s"
    dtype = "bf16"
    bound = "tensor"

    def __init__(self, size=16384):
        self.n = size
        self.name = f"gemm_splitk_{size}"

    def config(self, world):
        how = ("NCCL reduce-scatter of the fp32 partials + bias/tanh-GELU epilogue" if world > 1
               else "one rank: its partial is the sum, so afg_gemm_splitk runs the fused-epilogue "
                    "GEMM (no fp32 round trip, no collective)")
        return {"workload": f"bf16 matmul {self.n}^3 split-K over {world} rank(s), {how}",
                "M": self.n, "N": self.n, "K": self.n, "parallelism": f"splitK/{world}",
                "l2": "operands larger than L2"}

    def setup(self, rank, world, dev):
        import torch

        import oracle
        from paper_2603_06731_b200 import ops
        from paper_2603_06731_b200.tp import Comm, split_plan
        self.torch, self.ops = torch, ops
        n = self.n
        (k0, k1), _ = split_plan(n, n, rank, world)
        self.kl = k1 - k0
        self.A = ops.fill_uniform((n, self.kl), oracle.stream_seed("%a", 1 + rank), -1, 1,
                                  torch.bfloat16)
        self.B = ops.fill_uniform((self.kl, n), oracle.stream_seed("%b", 1 + rank), -1, 1,
                                  torch.bfloat16)
        self.bias = ops.fill_uniform((n,), oracle.stream_seed("%bias", 1), -1, 1, torch.float32)
        self.comm = Comm.from_process_group()
        self.C = torch.empty((n // world, n), dtype=torch.bfloat16, device=dev)
        from paper_2603_06731_b200 import lib
        ws = lib().afg_gemm_splitk_workspace(n, n, world, 0)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.flops_rank = 2.0 * n * n * self.kl
        self.flops_total = 2.0 * n ** 3
        self.alg_bytes_rank = 2.0 * (n * self.kl * 2 + n * n // world) + 4.0 * n * n

    def step(self):
        from paper_2603_06731_b200 import Epilogue
        from paper_2603_06731_b200.tp import gemm_splitk
        gemm_splitk(self.A, self.B, self.comm, bias=self.bias, epilogue=Epilogue.BIAS_GELU_TANH,
                    out=self.C, workspace=self.ws)

    def launches_per_step(self):
        return 2

    def e2e_setup(self):
        t = self.torch
        self.hA, self.hB = self.A.cpu().pin_memory(), self.B.cpu().pin_memory()
        self.hC = t.empty_like(self.C, device="cpu").pin_memory()
        self.h2d = (self.hA.numel() + self.hB.numel()) * 2
        self.d2h = self.hC.numel() * 2

    def e2e_step(self):
        self.A.copy_(self.hA, non_blocking=True)
        self.B.copy_(self.hB, non_blocking=True)
        self.step()
        self.hC.copy_(self.C, non_blocking=True)

    def reference_sample(self, threads):
        return ReferenceGemmSample(self.n, threads)


class GemmI8:
    """SURVEY 8f3 (beyond the BASELINE configs): the quant module's int8 GEMM
    (SPEC.md:531-572), i8 x i8 -> exact i32 accumulation, requantised to i8
    (round half away from zero, saturating), tcgen05 kind::i8."""

    metric = "TOP/s"
    unit = "TOP/s"
    dtype = "int8"
    bound = "tensor-i8"

    def __init__(self, size):
        self.n = size
        self.name = f"gemm_i8_{size}"

    def config(self, world):
        return {"workload": f"int8 matmul {self.n}x{self.n}x{self.n}, i32 accumulate, requantised "
                            f"i8 output (scale 2^-12), row-sharded",
                "M": self.n, "N": self.n, "K": self.n, "parallelism": f"rows/{world}",
                "l2": "operands larger than L2 (no flush needed)"}

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import ops
        self.torch, self.ops = torch, ops
        r0, r1 = shard_rows(self.n, rank, world)
        self.m = r1 - r0
        g = torch.Generator(device=dev).manual_seed(1000 + r0)
        self.A = torch.randint(-128, 128, (self.m, self.n), generator=g, dtype=torch.int8, device=dev)
        g.manual_seed(2)
        self.B = torch.randint(-128, 128, (self.n, self.n), generator=g, dtype=torch.int8, device=dev)
        self.C = torch.empty((self.m, self.n), dtype=torch.int8, device=dev)
        self.flops_rank = 2.0 * self.m * self.n * self.n
        self.flops_total = 2.0 * self.n ** 3
        self.alg_bytes_rank = float(self.m * self.n + self.n * self.n + self.m * self.n)

    def step(self):
        self.ops.gemm_i8(self.A, self.B, out_mode=1, scale=2.0 ** -12, out=self.C)

    def launches_per_step(self):
        return 1

    def e2e_setup(self):
        t = self.torch
        self.hA = self.A.cpu().pin_memory()
        self.hB = self.B.cpu().pin_memory()
        self.hC = t.empty((self.m, self.n), dtype=t.int8).pin_memory()
        self.dA = t.empty_like(self.A)
        self.dB = t.empty_like(self.B)
        self.h2d = self.hA.numel() + self.hB.numel()
        self.d2h = self.hC.numel()

    def e2e_step(self):
        self.dA.copy_(self.hA, non_blocking=True)
        self.dB.copy_(self.hB, non_blocking=True)
        self.ops.gemm_i8(self.dA, self.dB, out_mode=1, scale=2.0 ** -12, out=self.C)
        self.hC.copy_(self.C, non_blocking=True)

    def reference_sample(self, threads):
        return ReferenceI8Sample(self.n, threads)


class GemmFP32:
    """BASELINE configs[0]: fp32 1024^3 + bias + ReLU (replicas only)."""

    name = "gemm_fp32_relu"
    metric = "TFLOP/s"
    unit = "TFLOP/s"
    dtype = "f32"
    bound = "fp32-simt"

    def __init__(self, size=1024):
        self.n = size

    def config(self, world):
        return {"workload": f"fp32 matmul {self.n}^3 + bias + ReLU (the reference's own "
                            f"operator test), bit-exact vs af::interpret",
                "parallelism": f"replicas/{world}", "l2": "L2 flushed between steps (256 MB write + 256 MB read, untimed)"}

    def setup(self, rank, world, dev):
        import torch

        import oracle
        from paper_2603_06731_b200 import ops
        self.torch, self.ops = torch, ops
        n = self.n
        self.A = ops.fill_uniform((n, n), oracle.stream_seed("%a", 1), -1, 1, torch.float32)
        self.B = ops.fill_uniform((n, n), oracle.stream_seed("%b", 2), -1, 1, torch.float32)
        self.bias = ops.fill_uniform((n,), oracle.stream_seed("%bias", 3), -1, 1, torch.float32)
        self.C = torch.empty((n, n), dtype=torch.float32, device=dev)
        self.flush = L2Flush(dev)
        self.flops_rank = self.flops_total = 2.0 * n ** 3
        self.alg_bytes_rank = 4.0 * 3 * n * n

    def pre_step(self):
        self.flush()  # > L2: evict operands between steps (untimed)

    def step(self):
        from paper_2603_06731_b200 import Epilogue
        self.ops.gemm(self.A, self.B, bias=self.bias, epilogue=Epilogue.BIAS_RELU, out=self.C)

    def launches_per_step(self):
        return 1

    def e2e_setup(self):
        t = self.torch
        self.hA, self.hB = self.A.cpu().pin_memory(), self.B.cpu().pin_memory()
        self.hbias = self.bias.cpu().pin_memory()
        self.hC = t.empty_like(self.C, device="cpu").pin_memory()
        self.dA, self.dB, self.dbias = t.empty_like(self.A), t.empty_like(self.B), t.empty_like(self.bias)
        self.h2d = (self.hA.numel() + self.hB.numel() + self.hbias.numel()) * 4
        self.d2h = self.hC.numel() * 4

    def e2e_step(self):
        from paper_2603_06731_b200 import Epilogue
        self.dA.copy_(self.hA, non_blocking=True)
        self.dB.copy_(self.hB, non_blocking=True)
        self.dbias.copy_(self.hbias, non_blocking=True)
        self.ops.gemm(self.dA, self.dB, bias=self.dbias, epilogue=Epilogue.BIAS_RELU, out=self.C)
        self.hC.copy_(self.C, non_blocking=True)

    def reference_sample(self, threads):
        return ReferenceGemmSample(self.n, threads, act="relu", rows=8, cols=128)


class _Base:
    """Shared e2e plumbing: `self.host_inputs` (device tensor -> pinned host
    copy) are copied H2D every e2e step, `self.outputs` copied back D2H."""

    metric = "TFLOP/s"
    unit = "TFLOP/s"
    bound = "tensor"

    def launches_per_step(self):
        return 1

    def e2e_setup(self):
        t = self.torch
        self._h = [(d, d.cpu().pin_memory()) for d in self.e2e_inputs()]
        self._o = [(d, t.empty_like(d, device="cpu").pin_memory()) for d in self.e2e_outputs()]
        self.h2d = sum(h.numel() * h.element_size() for _, h in self._h)
        self.d2h = sum(h.numel() * h.element_size() for _, h in self._o)

    def e2e_step(self):
        for d, h in self._h:
            d.copy_(h, non_blocking=True)
        if getattr(self, "pre_step", None):
            self.pre_step()
        self.step()
        for d, h in self._o:
            h.copy_(d, non_blocking=True)


def _dev_uniform(shape, name, seed, lo, hi, dtype):
    import oracle

    from paper_2603_06731_b200 import ops
    return ops.fill_uniform(shape, oracle.stream_seed("%" + name, seed), lo, hi, dtype)


class Attention(_Base):
    """BASELINE configs[2]: fused attention fp16 B8 H16 S2048 D128, head-sharded."""

    dtype = "f16"

    def __init__(self, causal, B=8, H=16, S=2048, D=128):
        self.causal, self.B, self.H, self.S, self.D = causal, B, H, S, D
        self.name = "attention_causal" if causal else "attention"

    def config(self, world):
        return {"workload": f"fused attention fp16 B{self.B} H{self.H} S{self.S} D{self.D} "
                            f"{'causal' if self.causal else 'non-causal'}, scale 1/sqrt(D)",
                "parallelism": f"heads/{world}", "l2": "Q,K,V,O 268 MB > L2"}

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import ops
        self.torch, self.ops = torch, ops
        h0, h1 = shard_rows(self.B * self.H, rank, world)
        self.bh = h1 - h0
        shp = (1, self.bh, self.S, self.D)
        self.q = _dev_uniform(shp, "q", 1 + rank, -1, 1, torch.float16)
        self.k = _dev_uniform(shp, "k", 1 + rank, -1, 1, torch.float16)
        self.v = _dev_uniform(shp, "v", 1 + rank, -1, 1, torch.float16)
        self.o = torch.empty_like(self.q)
        f = 4.0 * self.S * self.S * self.D * (0.5 if self.causal else 1.0)
        self.flops_rank = f * self.bh
        self.flops_total = f * self.B * self.H
        self.alg_bytes_rank = 4.0 * self.bh * self.S * self.D * 2

    def step(self):
        self.ops.attention(self.q, self.k, self.v, scale=self.D ** -0.5, causal=self.causal,
                           out=self.o)

    def e2e_inputs(self):
        return [self.q, self.k, self.v]

    def e2e_outputs(self):
        return [self.o]

    def reference_sample(self, threads):
        return ReferenceGraphSample("attention", threads, causal=self.causal)


class GraphAPIGemm(_Base):
    """The drop-in path end to end: BASELINE configs[1]'s pattern written in
    the reference's unchanged graph API (matmul -> broadcast_in_dim(bias) ->
    add -> the 14-nest tanh-GELU composite, bf16 values in f32 tensors, SURVEY
    App. B) run through afg_graph_run exactly as a caller of af::interpret
    would: host doubles in, host doubles out, every step (parse, validate,
    device-verified pattern match, narrowing, the fused tcgen05 GEMM,
    download). Timed on the host clock (the step includes host work by
    definition); value = the GEMM's flops / step time."""

    dtype = "bf16"
    bound = "tensor"

    def __init__(self, n=4096):
        self.n = n
        self.name = f"graph_api_gemm_gelu_{n}"

    def config(self, world):
        return {"workload": f"reference graph API: {self.n}^3 matmul + bias + 14-nest GELU "
                            f"composite via afg_graph_run (host doubles in/out)",
                "parallelism": f"replicas/{world}", "l2": "n/a (host-side step)"}

    def setup(self, rank, world, dev):
        import torch

        import oracle as O
        from oracle.graphs import matmul_epi_graph
        self.torch = torch
        n = self.n
        g, fixed = matmul_epi_graph(n, n, n, "gelu")
        self.graph = json.dumps(g)
        self.inputs = {"a": O.round_to(O.random_tensor((n, n), "%a", 1, -1, 1), O.BF16),
                       "b": O.round_to(O.random_tensor((n, n), "%b", 1, -1, 1), O.BF16),
                       "bias": O.random_tensor((n,), "%bias", 1, -1, 1)}
        self.inputs.update(fixed)
        self.flops_rank = self.flops_total = 2.0 * n ** 3
        self.alg_bytes_rank = 8.0 * 3 * n * n

    def step(self):
        from paper_2603_06731_b200.graph import execute
        self.out, self.plan = execute(self.graph, self.inputs, want_plan=True)

    def e2e_setup(self):
        self.h2d = sum(v.size * 8 for v in self.inputs.values())
        self.d2h = self.n * self.n * 8

    def e2e_step(self):
        self.step()

    def reference_sample(self, threads):
        return ReferenceGemmSample(self.n, threads)


def measure_host(ctx, wl, steps):
    """Host-clock timing for host-side steps (the graph API path)."""
    wl.setup(ctx.rank, ctx.world, ctx.dev)
    wl.step()
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        wl.step()
    ctx.barrier()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    ms_max = ctx.max_over_ranks(ms)
    value = wl.flops_total / (ms_max * 1e-3) / 1e12
    return {"value": value, "unit": "TFLOP/s", "ms_per_step": ms_max, "steps": steps,
            "dtype": wl.dtype, "timing": "host clock (the step is host-side by definition)",
            "plan": getattr(wl, "plan", None), "workload": wl.config(ctx.world)["workload"]}


# ResNet-50 (v1.5) 3x3 / 1x1 conv layers: (H_in, C, OC, k, stride, count), BASELINE.md §5
RESNET50 = [(56, 64, 64, 1, 1, 1), (56, 64, 64, 3, 1, 3), (56, 64, 256, 1, 1, 3),
            (56, 64, 256, 1, 1, 1), (56, 256, 64, 1, 1, 2), (56, 256, 128, 1, 1, 1),
            (56, 128, 128, 3, 2, 1), (28, 128, 128, 3, 1, 3), (28, 128, 512, 1, 1, 4),
            (56, 256, 512, 1, 2, 1), (28, 512, 128, 1, 1, 3), (28, 512, 256, 1, 1, 1),
            (28, 256, 256, 3, 2, 1), (14, 256, 256, 3, 1, 5), (14, 256, 1024, 1, 1, 6),
            (28, 512, 1024, 1, 2, 1), (14, 1024, 256, 1, 1, 5), (14, 1024, 512, 1, 1, 1),
            (14, 512, 512, 3, 2, 1), (7, 512, 512, 3, 1, 2), (7, 512, 2048, 1, 1, 3),
            (14, 1024, 2048, 1, 2, 1), (7, 2048, 512, 1, 1, 2)]


class ResNetConvs(_Base):
    """BASELINE configs[3]: all ResNet-50 3x3/1x1 convs (53 launches, 2.03 TFLOP
    at batch 256), NHWC bf16 implicit GEMM + bias + ReLU, batch-sharded."""

    dtype = "bf16"
    name = "resnet50_convs"

    def __init__(self, batch=256):
        self.batch = batch

    def config(self, world):
        return {"workload": f"ResNet-50 3x3/1x1 conv layers (23 shapes, 53 convs), NHWC bf16 "
                            f"implicit GEMM + bias + ReLU, batch {self.batch}",
                "parallelism": f"batch/{world}", "l2": "activations > L2 for the 56x56 layers"}

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import ops
        self.torch, self.ops = torch, ops
        b0, b1 = shard_rows(self.batch, rank, world)
        self.b = b1 - b0
        self.layers = []
        self.ops_fb = []  # (count, flops, bytes) per layer: the per-layer roofline floor
        self.flops_rank = 0.0
        self.alg_bytes_rank = 0.0
        for i, (H, C, OC, k, s, cnt) in enumerate(RESNET50):
            pad = 1 if k == 3 else 0
            OH = (H + 2 * pad - k) // s + 1
            x = _dev_uniform((self.b, H, H, C), f"x{i}", 1, -1, 1, torch.bfloat16)
            w = _dev_uniform((OC, k, k, C), f"w{i}", 1, -0.1, 0.1, torch.bfloat16)
            bias = _dev_uniform((OC,), f"b{i}", 1, -1, 1, torch.float32)
            y = torch.empty((self.b, OH, OH, OC), dtype=torch.bfloat16, device=dev)
            self.layers.append((x, w, bias, y, k, s, pad, cnt))
            # a strided 1x1 conv reads only every s-th pixel of its input
            x_read = self.b * OH * OH * C if (k == 1 and s > 1) else x.numel()
            self.flops_rank += cnt * 2.0 * self.b * OH * OH * OC * C * k * k
            self.alg_bytes_rank += cnt * 2.0 * (x_read + y.numel() + w.numel())
            self.ops_fb.append((cnt, 2.0 * self.b * OH * OH * OC * C * k * k,
                                2.0 * (x_read + y.numel() + w.numel())))
        self.flops_total = self.flops_rank * self.batch / self.b

    def step(self):
        from paper_2603_06731_b200 import Epilogue, check, lib
        import ctypes
        L = lib()
        st = ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)
        for x, w, bias, y, k, s, pad, cnt in self.layers:
            B, H, W, C = x.shape
            OC, OH = w.shape[0], y.shape[1]
            for _ in range(cnt):
                check(L.afg_conv2d_nhwc(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(),
                                        B, H, W, C, OC, k, k, s, s, pad, pad, 1, 1, OH, OH, 2,
                                        int(Epilogue.BIAS_RELU), st))

    def launches_per_step(self):
        return sum(l[-1] for l in self.layers)

    def e2e_inputs(self):
        return [l[0] for l in self.layers]

    def e2e_outputs(self):
        return [l[3] for l in self.layers]

    def reference_sample(self, threads):
        return ReferenceGraphSample("conv", threads)


class BertLayer(_Base):
    """BASELINE configs[4]: BERT-base encoder layer, B64 x S512, bf16,
    batch-sharded (afg_encoder_layer_fwd: 7 launches)."""

    dtype = "bf16"
    name = "bert_layer"

    def __init__(self, batch=64, seq=512, hidden=768, heads=12, ffn=3072):
        self.batch, self.seq, self.hd, self.heads, self.ffn = batch, seq, hidden, heads, ffn

    def config(self, world):
        return {"workload": f"BERT-base encoder layer (QKV GEMM, fused attention, out-proj+"
                            f"residual, LN, GELU FFN, LN) B{self.batch} x S{self.seq}, bf16",
                "parallelism": f"batch/{world}", "l2": "activations 50 MB-200 MB per op"}

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import lib
        self.torch = torch
        b0, b1 = shard_rows(self.batch, rank, world)
        self.b = b1 - b0
        T, hd, ffn = self.b * self.seq, self.hd, self.ffn
        bf, f32 = torch.bfloat16, torch.float32
        self.x = _dev_uniform((T, hd), "x", 1, -1, 1, bf)
        self.y = torch.empty_like(self.x)
        self.w = {"qkv": _dev_uniform((hd, 3 * hd), "wqkv", 1, -0.05, 0.05, bf),
                  "o": _dev_uniform((hd, hd), "wo", 1, -0.05, 0.05, bf),
                  "1": _dev_uniform((hd, ffn), "w1", 1, -0.05, 0.05, bf),
                  "2": _dev_uniform((ffn, hd), "w2", 1, -0.05, 0.05, bf)}
        self.p = {"bqkv": _dev_uniform((3 * hd,), "bqkv", 1, -0.1, 0.1, f32),
                  "bo": _dev_uniform((hd,), "bo", 1, -0.1, 0.1, f32),
                  "g1": _dev_uniform((hd,), "g1", 1, 0.9, 1.1, f32),
                  "be1": _dev_uniform((hd,), "be1", 1, -0.1, 0.1, f32),
                  "b1": _dev_uniform((ffn,), "b1", 1, -0.1, 0.1, f32),
                  "b2": _dev_uniform((hd,), "b2", 1, -0.1, 0.1, f32),
                  "g2": _dev_uniform((hd,), "g2", 1, 0.9, 1.1, f32),
                  "be2": _dev_uniform((hd,), "be2", 1, -0.1, 0.1, f32)}
        self.ws_bytes = lib().afg_encoder_layer_workspace(self.b, self.seq, hd, ffn, 2)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        gemm = 2.0 * T * hd * (3 * hd + hd + 2 * ffn)
        attn = 4.0 * self.b * self.heads * self.seq * self.seq * (hd // self.heads)
        # (count, flops, bytes) per launch: the per-op roofline floor (bf16 bytes)
        self.ops_fb = [(1, 2.0 * T * hd * 3 * hd, 2.0 * (T * hd + 3 * hd * hd + 3 * T * hd)),
                       (1, attn, 2.0 * (3 * T * hd + T * hd)),
                       (1, 2.0 * T * hd * hd, 2.0 * (T * hd + hd * hd + 2 * T * hd)),
                       (2, 0.0, 2.0 * 3 * T * hd),
                       (1, 2.0 * T * hd * ffn, 2.0 * (T * hd + hd * ffn + T * ffn)),
                       (1, 2.0 * T * ffn * hd, 2.0 * (T * ffn + ffn * hd + 2 * T * hd))]
        self.flops_rank = gemm + attn
        self.flops_total = self.flops_rank * self.batch / self.b
        self.alg_bytes_rank = 2.0 * T * hd * 2

    def step(self):
        import ctypes

        from paper_2603_06731_b200 import check, lib
        L = lib()
        p, w = self.p, self.w
        st = ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)
        check(L.afg_encoder_layer_fwd(
            self.x.data_ptr(), self.y.data_ptr(), self.b, self.seq, self.hd, self.heads, self.ffn,
            w["qkv"].data_ptr(), p["bqkv"].data_ptr(), w["o"].data_ptr(), p["bo"].data_ptr(),
            p["g1"].data_ptr(), p["be1"].data_ptr(), w["1"].data_ptr(), p["b1"].data_ptr(),
            w["2"].data_ptr(), p["b2"].data_ptr(), p["g2"].data_ptr(), p["be2"].data_ptr(),
            1e-12, 2, self.ws.data_ptr(), self.ws_bytes, st))

    def launches_per_step(self):
        return 7

    def e2e_inputs(self):
        return [self.x]

    def e2e_outputs(self):
        return [self.y]

    def reference_sample(self, threads):
        return ReferenceGraphSample("bert", threads)


class MemChain(_Base):
    """Memory-bound chains (K4 softmax fp16 [8*16*2048, 2048]; K5 residual +
    layernorm bf16 [32768, 768]); metric GB/s of algorithmic bytes."""

    metric = "GB/s"
    unit = "GB/s"
    bound = "hbm"

    def __init__(self, kind):
        self.kind = kind
        self.name = kind
        self.dtype = "f16" if kind == "softmax" else "bf16"

    def config(self, world):
        what = ("row softmax fp16 [262144, 2048]" if self.kind == "softmax" else
                "residual + layernorm bf16 [32768, 768] (x + r -> y, fp32 stats)")
        return {"workload": what, "parallelism": f"rows/{world}",
                "l2": "inputs larger than L2" if self.kind == "softmax" else
                "L2 flushed between steps (256 MB write + 256 MB read, untimed)"}

    def setup(self, rank, world, dev):
        import torch

        from paper_2603_06731_b200 import ops
        self.torch, self.ops = torch, ops
        if self.kind == "softmax":
            rows, cols, dt = 8 * 16 * 2048, 2048, torch.float16
        else:
            rows, cols, dt = 32768, 768, torch.bfloat16
        r0, r1 = shard_rows(rows, rank, world)
        n = r1 - r0
        self.x = _dev_uniform((n, cols), "x", 1, -4, 4, dt)
        self.y = torch.empty_like(self.x)
        self.flush = None
        if self.kind == "layernorm":
            self.r = _dev_uniform((n, cols), "r", 1, -1, 1, dt)
            self.g = _dev_uniform((cols,), "g", 1, 0.9, 1.1, torch.float32)
            self.b = _dev_uniform((cols,), "b", 1, -0.1, 0.1, torch.float32)
            self.flush = L2Flush(dev)
            self.alg_bytes_rank = 3.0 * n * cols * 2
        else:
            self.alg_bytes_rank = 2.0 * n * cols * 2
        self.flops_rank = self.alg_bytes_rank
        self.flops_total = self.alg_bytes_rank * rows / n

    def pre_step(self):
        if self.flush is not None and not os.environ.get("AFG_BENCH_NO_FLUSH"):
            self.flush()  # untimed L2 flush (the LN working set fits in L2)

    def step(self):
        if self.kind == "softmax":
            self.ops.softmax(self.x, out=self.y)
        else:
            self.ops.layernorm_residual(self.x, self.r, self.g, self.b, out=self.y)

    def e2e_inputs(self):
        return [self.x] + ([self.r] if self.kind == "layernorm" else [])

    def e2e_outputs(self):
        return [self.y]

    def reference_sample(self, threads):
        return ReferenceGraphSample("softmax", threads)


WORKLOADS = {"gemm_bf16": lambda a: GemmBF16(a.size), "gemm_fp32": lambda a: GemmFP32(),
             "gemm_splitk": lambda a: GemmSplitK(a.size),
             "gemm_i8": lambda a: GemmI8(a.size),
             "attention": lambda a: Attention(False), "attention_causal": lambda a: Attention(True),
             "resnet50_convs": lambda a: ResNetConvs(), "bert_layer": lambda a: BertLayer(),
             "softmax": lambda a: MemChain("softmax"), "layernorm": lambda a: MemChain("layernorm")}


# ======================================================= reference path ===

def gemm_graph(m, n, k, act):
    """matmul -> broadcast_in_dim(bias) -> add -> act in the unchanged graph
    API (GELU = the 14-nest composite)."""
    from oracle.graphs import matmul_epi_graph
    g, fixed = matmul_epi_graph(m, n, k, act)
    return g, fixed


class ReferenceGemmSample:
    """One bounded sample of the GEMM workload through the reference's CPU
    path: af::lowerGraphToAffine + af::interpret (oracle/_ref), one
    independent interpreter instance per host thread on its own
    [rows x K] x [K x cols] shard (the interpreter is single-threaded and
    safe across instances). Falls back to the oracle C port
    (kind "port") when the reference build is absent."""

    def __init__(self, K, threads, act="gelu", rows=2, cols=32):
        import oracle as O
        self.O = O
        self.K, self.threads, self.rows, self.cols = K, threads, rows, cols
        self.kind = "reference" if O.ref_available() else "port"
        g, fixed = gemm_graph(rows, cols, K, act)
        self.graph = json.dumps(g)
        self.inputs = O.random_graph_inputs(g, 7, -1.0, 1.0)
        self.inputs.update(fixed)
        self.act = act
        self.flops = 2.0 * rows * cols * K * threads

    def describe(self):
        how = ("af::lowerGraphToAffine + af::interpret (AffineForge reference, oracle/_ref)"
               if self.kind == "reference" else "oracle C port (interp semantics)")
        return (f"{self.threads} independent shards of [{self.rows}x{self.K}]x[{self.K}x{self.cols}]"
                f" matmul+bias+{self.act} via {how}")

    def run_once(self):
        from concurrent.futures import ThreadPoolExecutor
        O = self.O

        def one(_):
            if self.kind == "reference":
                O.ref_run(self.graph, self.inputs, "interpret")
            else:
                ins = {k: O.round_to(v, O.F32) for k, v in self.inputs.items()}
                epi = O.EPI_GELU_TANH if self.act == "gelu" else O.EPI_RELU
                O.matmul(ins["a"], ins["b"], ins["bias"], epi=epi, interp=True, nthreads=1)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(one, range(self.threads)))
        return time.perf_counter() - t0


class ReferenceI8Sample:
    """Bounded reference-path sample of the int8 GEMM: one af::interpret
    instance per host thread on an i8 [rows x K] x [K x cols] -> i32 matmul
    graph (the oracle's integer restatement when oracle/_ref is absent)."""

    def __init__(self, K, threads, rows=2, cols=32):
        import oracle as O
        self.O, self.K, self.threads, self.rows, self.cols = O, K, threads, rows, cols
        self.kind = "reference" if O.ref_available() else "port"
        rng = np.random.default_rng(7)
        self.a = rng.integers(-128, 128, (rows, K))
        self.b = rng.integers(-128, 128, (K, cols))
        self.graph = json.dumps({
            "tensors": [{"id": "a", "shape": [rows, K], "dtype": "i8"},
                        {"id": "b", "shape": [K, cols], "dtype": "i8"},
                        {"id": "c", "shape": [rows, cols], "dtype": "i32"}],
            "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]})
        self.flops = 2.0 * rows * cols * K * threads

    def describe(self):
        how = "af::interpret (oracle/_ref)" if self.kind == "reference" else "oracle integer port"
        return (f"{self.threads} independent shards of i8 [{self.rows}x{self.K}]x[{self.K}x"
                f"{self.cols}] -> i32 matmul via {how}")

    def run_once(self):
        from concurrent.futures import ThreadPoolExecutor
        O = self.O

        def one(_):
            if self.kind == "reference":
                O.ref_run(self.graph, {"a": self.a, "b": self.b}, "interpret")
            else:
                O.matmul_i8(self.a, self.b.T)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(one, range(self.threads)))
        return time.perf_counter() - t0


class ReferenceGraphSample:
    """Bounded reference-path sample for the non-GEMM workloads: one
    af::interpret instance per host thread on a small instance of the same op
    graph (attention: one head at N=64, D=128; conv: 3x3 64->64 on 8x8;
    softmax: 64 rows x 2048), metric units as the workload's."""

    def __init__(self, kind, threads, causal=False):
        import oracle as O
        from oracle.graphs import attention_graph, nhwc_conv_graph, T
        self.O, self.kind, self.threads = O, kind, threads
        self.kindref = "reference" if O.ref_available() else "port"
        if kind == "attention":
            N, D = 64, 128
            g, fixed = attention_graph(1, 1, N, D, causal)
            self.flops = 4.0 * N * N * D * (0.5 if causal else 1.0) * threads
            self.desc = f"1 head N={N} D={D} attention graph"
        elif kind == "bert":
            from oracle.graphs import bert_layer_graph
            g, fixed, fl = bert_layer_graph(32, 64, 2, 256)
            self.flops = fl * threads
            self.desc = ("BERT encoder layer graph S=32 hidden=64 heads=2 ffn=256 (QKV/out/FFN "
                         "matmuls + bias, scaled attention, GELU composite, residuals; LN has "
                         "no reference op)")
        elif kind == "conv":
            g, fixed = nhwc_conv_graph(1, 8, 8, 64, 64, 3, 1, "same")
            self.flops = 2.0 * 64 * 64 * 64 * 9 * threads
            self.desc = "3x3 64->64 NHWC conv graph on 1x8x8"
        else:
            g = {"tensors": [T("x", [64, 2048], "f16"), T("y", [64, 2048], "f16")],
                 "ops": [{"op": "softmax", "inputs": ["x"], "output": "y", "attrs": {"axis": -1}}]}
            fixed = {}
            self.flops = 2.0 * 64 * 2048 * 2 * threads  # bytes, for the GB/s metric
            self.desc = "softmax f16 64x2048 graph"
        self.graph = json.dumps(g)
        self.inputs = O.random_graph_inputs(g, 7, -1.0, 1.0)
        self.inputs.update(fixed)
        self.kind_graph = g

    @property
    def kind_label(self):
        return self.kindref

    def describe(self):
        return (f"{self.threads} independent af::interpret instances, each a {self.desc}"
                if self.kindref == "reference" else f"{self.threads} x {self.desc} via oracle port")

    def run_once(self):
        from concurrent.futures import ThreadPoolExecutor
        O = self.O

        def one(_):
            if self.kindref == "reference":
                O.ref_run(self.graph, self.inputs, "interpret")
            elif self.kind == "attention":
                ins = self.inputs
                O.attention(ins["q"], ins["k"], ins["v"], nthreads=1)
            elif self.kind == "conv":
                ins = self.inputs
                O.conv_nhwc(ins["x"], np.transpose(ins["w"], (0, 2, 3, 1)), ins["bias"], (1, 1),
                            (1, 1), epi=O.EPI_RELU, nthreads=1)
            else:
                O.softmax(self.inputs["x"])
        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(one, range(self.threads)))
        return time.perf_counter() - t0


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, wl, rank, world):
    """--impl reference: the reference CPU path on the host cores."""
    if rank != 0:
        return 0
    threads = host_threads()
    sample = wl.reference_sample(threads)
    for _ in range(args.warmup):
        sample.run_once()
    times = [sample.run_once() for _ in range(args.steps)]
    t = sum(times) / len(times)
    value = sample.flops / t / (1e9 if wl.unit == "GB/s" else 1e12)
    line = {"metric": wl.metric, "value": value, "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak" if isinstance(wl, GemmFP32) else "strong",
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic (makeRandomTensor)",
            "config": wl.config(world), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": wl.unit, "cores": threads,
                             "kind": getattr(sample, "kind_label", getattr(sample, "kind", None)),
                             "sample": sample.describe()},
            "e2e": {"value": value, "unit": wl.unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ============================================================== afg arm ===

class Ctx:
    """Per-process device / distributed plumbing shared by every workload."""

    def __init__(self, rank, world, local):
        import torch
        self.torch = torch
        self.rank, self.world, self.local = rank, world, local
        self.dev = torch.device(f"cuda:{local}")
        torch.cuda.set_device(self.dev)
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=self.dev)
        self.peaks = load_peaks()

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, v):
        if self.world == 1:
            return v
        import torch.distributed as dist
        t = self.torch.tensor([v], device=self.dev, dtype=self.torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


def measure(ctx, wl, steps, warmup, no_graph=False, min_timed_s=0.25):
    """Device-timed steps of one workload: W warm-up steps, the step captured
    once into a CUDA graph and replayed, K timed steps (at least `min_timed_s`
    of device time so the clock sampler sees the region), each bracketed by
    CUDA events on the launching stream, barrier + sync on both sides, the
    mean step time max-reduced over ranks. Returns the measurement dict."""
    import torch

    import paper_2603_06731_b200 as afg
    wl.setup(ctx.rank, ctx.world, ctx.dev)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    pre = getattr(wl, "pre_step", None)  # untimed per-step prologue (L2 flush)
    t0 = time.perf_counter()
    for _ in range(max(warmup, 3)):
        if pre:
            pre()
        wl.step()
    torch.cuda.synchronize()
    est = (time.perf_counter() - t0) / max(warmup, 3)
    steps = max(steps, min(200, int(math.ceil(min_timed_s / max(est, 1e-5)))))
    run = wl.step
    graph = None
    launches_per_step = None
    if not no_graph:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            wl.step()
        stream.wait_stream(side)
        torch.cuda.synchronize()
        launches0 = afg.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            wl.step()
        run = graph.replay
        launches_per_step = afg.launch_count() - launches0
    for _ in range(2):
        if pre:
            pre()
        run()
    ctx.barrier()
    clocks = ClockSampler(ctx.local)
    clocks.start()
    time.sleep(0.3)
    launches0 = afg.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    ctx.barrier()
    # hold the GPU in a ~2 ms spin before the first step so the host enqueues
    # every step (graph replays, events) ahead of the device: no host launch
    # latency can sit between a step's start and end events
    torch.cuda._sleep(4_000_000)
    for i in range(steps):
        if pre:
            pre()  # enqueued before the start event: the GPU is busy, timing is exact
        evs[i][0].record(stream)
        run()
        evs[i][1].record(stream)
    ctx.barrier()
    launches = (launches_per_step * steps if graph is not None
                else afg.launch_count() - launches0)
    step_ms = [x.elapsed_time(y) for x, y in evs]
    ms = sum(step_ms) / steps  # ONE statistic (the mean) for value and roofline
    clk = clocks.stop()
    ms_max = ctx.max_over_ranks(ms)
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    value = wl.flops_total / (ms_max * 1e-3) / scale
    peaks = ctx.peaks
    peak_note = f"{peaks['source']} (MEASURED_PEAKS.json burst)"
    bound = wl.bound
    if bound == "hbm":
        achieved = wl.alg_bytes_rank / (ms * 1e-3) / 1e9
        peak, unit = peaks["hbm_gbs"], "GB/s"
    elif bound == "tensor-i8":  # dense int8 = 2x dense bf16 on B200 (4.5 vs 2.25 PFLOP/s nominal)
        achieved = wl.flops_rank / (ms * 1e-3) / 1e12
        peak, unit = 2.0 * peaks["bf16_tflops"], "TOP/s"
        peak_note = (f"assumed: 2 x the {peaks['source']} bf16 burst peak (MEASURED_PEAKS.json "
                     f"has no int8 entry; nominal dense int8 = 2 x dense bf16)")
    elif bound == "fp32-simt":
        achieved = wl.flops_rank / (ms * 1e-3) / 1e12
        peak, unit = fp32_simt_peak(clk), "TFLOP/s"
        peak_note = ("derived FP32 CUDA-core peak: 148 SM x 128 lanes x 2 flop x sm_max_mhz "
                     "(the path is the interpreter-exact fp32 GEMM, no tensor cores)")
    else:
        achieved = wl.flops_rank / (ms * 1e-3) / 1e12
        peak, unit = peaks["bf16_tflops"], "TFLOP/s"
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "peak_source": peak_note, "step_ms": ms,
            "statistic": "mean of the timed steps (same as value)",
            "traffic": traffic_for(wl.name), **floor_fields(wl, peaks, ms)}
    if bound == "fp32-simt":
        roof["frac_of_bf16_peak"] = achieved / peaks["bf16_tflops"]
    return {"metric": wl.metric, "value": value, "unit": wl.unit, "ms_per_step": ms_max,
            "steps": steps, "dtype": wl.dtype, "config": wl.config(ctx.world), "roofline": roof,
            "gpu_launches": int(launches), "clocks": clk}


def measure_e2e(ctx, wl, steps):
    """The same metric end to end through the C ABI with pinned host buffers:
    every step copies its inputs H2D and its result D2H inside the timed
    region (device-timed, max over ranks)."""
    import torch
    stream = torch.cuda.current_stream()
    wl.e2e_setup()
    for _ in range(2):
        wl.e2e_step()
    ctx.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e_steps = max(1, min(steps, 5))
    e0.record(stream)
    for _ in range(e_steps):
        wl.e2e_step()
    e1.record(stream)
    ctx.barrier()
    e_ms = ctx.max_over_ranks(e0.elapsed_time(e1) / e_steps)
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    return {"value": wl.flops_total / (e_ms * 1e-3) / scale, "unit": wl.unit, "ms_per_step": e_ms,
            "h2d_bytes_per_step": wl.h2d * ctx.world, "d2h_bytes_per_step": wl.d2h * ctx.world,
            "path": getattr(wl, "e2e_path", "pinned host -> cudaMemcpyAsync -> afg C ABI -> D2H")}


def cpu_baseline(wl):
    threads = host_threads()
    sample = wl.reference_sample(threads)
    t = sample.run_once()
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    return {"value": sample.flops / t / scale, "unit": wl.unit, "cores": threads,
            "kind": getattr(sample, "kind_label", getattr(sample, "kind", None)),
            "sample": sample.describe(), "seconds": t}


def release(wl):
    import gc

    import torch
    if getattr(wl, "comm", None) is not None:
        torch.cuda.synchronize()
        wl.comm.close()
    for k in list(vars(wl)):
        if k not in ("torch", "ops"):
            setattr(wl, k, None)
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


# the other BASELINE configs measured in the default run (name, constructor)
SUB_WORKLOADS = [
    ("gemm_bf16_2048", lambda: GemmBF16(2048)), ("gemm_bf16_4096", lambda: GemmBF16(4096)),
    ("gemm_bf16_8192", lambda: GemmBF16(8192)), ("gemm_fp32_1024", lambda: GemmFP32()),
    ("attention", lambda: Attention(False)), ("attention_causal", lambda: Attention(True)),
    ("resnet50_convs", lambda: ResNetConvs()), ("bert_layer", lambda: BertLayer()),
    ("softmax", lambda: MemChain("softmax")), ("layernorm", lambda: MemChain("layernorm")),
    ("gemm_i8_8192", lambda: GemmI8(8192)), ("gemm_splitk_16384", lambda: GemmSplitK(16384)),
]


def run_afg(args, wl, rank, world, local, subs=()):
    ctx = Ctx(rank, world, local)
    m = measure(ctx, wl, args.steps, args.warmup, args.no_graph)
    e2e = measure_e2e(ctx, wl, args.steps)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)
    release(wl)
    workloads = {}
    if subs:  # the drop-in graph path, host doubles in / out (host-clock timed)
        g = GraphAPIGemm(4096)
        try:
            workloads["graph_api_gemm_gelu_4096"] = measure_host(ctx, g, 3)
        except Exception as e:
            workloads["graph_api_gemm_gelu_4096"] = {"error": f"{type(e).__name__}: {e}"}
        release(g)
    # each sub-workload starts after a short idle period so it does not inherit
    # the previous measurement's power / thermal state (the chip runs under its
    # power cap; back to back, later entries measured 5-10 % below their
    # stand-alone --only runs)
    cooldown = float(os.environ.get("AFG_BENCH_COOLDOWN_S", "3"))
    for name, make in subs:
        ctx.barrier()
        time.sleep(cooldown)
        sub = make()
        try:
            r = measure(ctx, sub, min(args.steps, 20), args.warmup, args.no_graph,
                        min_timed_s=0.15)
            workloads[name] = {k: r[k] for k in ("value", "unit", "ms_per_step", "steps",
                                                 "dtype", "roofline", "clocks", "gpu_launches")}
            workloads[name]["workload"] = r["config"].get("workload")
            workloads[name]["cooldown_s"] = cooldown
        except Exception as e:  # report, never hide: the entry says what failed
            workloads[name] = {"error": f"{type(e).__name__}: {e}"}
        release(sub)
    if rank == 0:
        line = {"metric": m["metric"], "value": m["value"], "unit": m["unit"], "n_gpus": world,
                "steps": m["steps"], "warmup": max(args.warmup, 3),
                "ms_per_step": m["ms_per_step"], "higher_is_better": True,
                "scaling": "weak" if isinstance(wl, GemmFP32) else "strong",
                "vs_baseline": None, "dtype": m["dtype"],
                "data": "synthetic (device-side makeRandomTensor stream, uniform)",
                "config": m["config"], "roofline": m["roofline"], "e2e": e2e,
                "gpu_launches": m["gpu_launches"], "clocks": m["clocks"],
                "cpu_baseline": cpu, "impl": "afg"}
        if workloads:
            line["workloads"] = workloads
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="afg", choices=["afg", "reference"])
    ap.add_argument("--workload", default="gemm_bf16", choices=sorted(WORKLOADS))
    ap.add_argument("--all", action="store_true", help="run every workload (one line each)")
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying "
                    "a captured CUDA graph of the step")
    ap.add_argument("--only", action="store_true", help="the named workload alone (no "
                    "'workloads' sub-dict in the default run)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    names = sorted(WORKLOADS) if args.all else [args.workload]
    default_run = (args.workload == "gemm_bf16" and args.size == 16384 and not args.all
                   and not args.only)
    for name in names:
        wl = WORKLOADS[name](args)
        if args.impl == "reference":
            run_reference(args, wl, rank, world)
        else:
            run_afg(args, wl, rank, world, local, SUB_WORKLOADS if default_run else ())
    return 0


if __name__ == "__main__":
    sys.exit(main())
