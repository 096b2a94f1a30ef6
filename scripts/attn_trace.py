"""Runs one attention launch with AFG_ATTN_TRACE=1 and summarises CTA 0's
timeline (clock64 cycles): per unit the S-ready -> P-written softmax time of
each tile, gaps between a tile's steps, and the unit-boundary gaps."""
import os
import subprocess
import sys

args = sys.argv[1:] or ["8", "16", "2048", "128", "0"]
code = f"""
import sys, torch
sys.path.insert(0, '.')
from paper_2603_06731_b200 import ops
B, H, N, D, causal = {args[0]}, {args[1]}, {args[2]}, {args[3]}, {args[4]}
q, k, v = (torch.rand(B, H, N, D, device='cuda').half() for _ in range(3))
ops.attention(q, k, v, scale=D ** -0.5, causal=bool(causal))
torch.cuda.synchronize()
"""
env = dict(os.environ, AFG_ATTN_TRACE="1")
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stderr
ev = []
for line in out.splitlines():
    if line.startswith("T "):
        kv = dict(x.split("=") for x in line[2:].split())
        ev.append({k: int(v) for k, v in kv.items()})
names = {1: "S_ready", 2: "P_done", 3: "O_ready", 4: "O_read", 5: "Q_ready(mma)", 6: "PV_A", 7: "PV_B",
         8: "Q_issue"}
for e in ev[:400]:
    print(f"{e['t']:>10} role{e['role']} {names.get(e['code'], e['code']):>12} u{e['unit']} j{e['step']}")
