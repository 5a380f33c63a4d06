"""Host-side cost of the e2e decode step (config B): time to enqueue the 32
ta_attend_host_async calls and the next step's ta_prepare, vs the step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_00242_b200 import TreeAttention
cfg = bench.CONFIGS["few_shot"]
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
ctx = TreeAttention(n_layers=32, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16)
ctx.restore(*snap)
L = len(ctx.leaves())
qh = torch.empty((32, L, 32, 128), dtype=torch.bfloat16).pin_memory()
oh = torch.empty_like(qh).pin_memory()
qn, on = qh.view(torch.int16).numpy(), oh.view(torch.int16).numpy()
s = torch.cuda.current_stream()
ctx.prepare(128, s)
for it in range(8):
    t0 = time.perf_counter()
    for layer in range(32):
        ctx.attend_host_async(layer, qn[layer], on[layer], stream=s)
    t1 = time.perf_counter()
    ctx.prepare(128, s)
    t2 = time.perf_counter()
    ctx.attend_host_wait()
    t3 = time.perf_counter()
    if it >= 3:
        print(f"enqueue 32 layers {1e6*(t1-t0):.0f} us, prepare {1e6*(t2-t1):.0f} us, wait {1e6*(t3-t2):.0f} us, step {1e6*(t3-t0):.0f} us")
