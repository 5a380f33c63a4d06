"""Host-side cost of the e2e path (debug): prepare, attend_host_async issue time per layer."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2404_00242_b200 import TreeAttention, capi

cfg = bench.CONFIGS["few_shot"]
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
n = 32
ctx = TreeAttention(n_layers=n, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16)
ctx.restore(*snap)
for layer in range(n):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c:
            ctx.write_kv(layer, int(node), (torch.rand((c, 8, 128), device="cuda") * 2 - 1).bfloat16(),
                         (torch.rand((c, 8, 128), device="cuda") * 2 - 1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((n, L, 32, 128)) * 2 - 1).bfloat16().pin_memory()
o = torch.empty((n, L, 32, 128), dtype=torch.bfloat16).pin_memory()
qn = q.view(torch.int16).numpy()
on = o.view(torch.int16).numpy()
s = torch.cuda.current_stream()
for _ in range(3):
    ctx.prepare(128, s)
    for l in range(n):
        ctx.attend_host_async(l, qn[l], on[l], stream=s)
    ctx.attend_host_wait()
T = {"prepare": 0.0, "issue": 0.0, "wait": 0.0}
R = 20
for _ in range(R):
    t0 = time.perf_counter()
    ctx.prepare(128, s)
    t1 = time.perf_counter()
    for l in range(n):
        ctx.attend_host_async(l, qn[l], on[l], stream=s)
    t2 = time.perf_counter()
    ctx.attend_host_wait()
    t3 = time.perf_counter()
    T["prepare"] += t1 - t0
    T["issue"] += t2 - t1
    T["wait"] += t3 - t2
print({k: round(v / R * 1e6, 1) for k, v in T.items()}, "us per step;", round(T["issue"] / R / n * 1e6, 2), "us per issue")
# raw ctypes cost of the issue call (no python wrapper)
lib = capi.lib()
import ctypes as C
qp = [C.c_void_p(qn[l].ctypes.data) for l in range(n)]
op = [C.c_void_p(on[l].ctypes.data) for l in range(n)]
sp = C.c_void_p(s.cuda_stream)
t0 = time.perf_counter()
for _ in range(R):
    ctx.prepare(128, s)
    for l in range(n):
        lib.ta_attend_host_async(ctx._h, l, qp[l], op[l], sp)
    ctx.attend_host_wait()
print("raw ctypes step", round((time.perf_counter() - t0) / R * 1e6, 1), "us")
