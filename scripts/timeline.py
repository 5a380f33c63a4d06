"""Per-launch timeline of consecutive layer calls (debug): first-CTA start /
last-CTA end of each attention launch and its merge launch (globaltimer, ns),
eager PDL-chained launches of n layers on one stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2404_00242_b200 import TreeAttention

name = sys.argv[1] if len(sys.argv) > 1 else "few_shot"
cfg = dict(bench.CONFIGS[name])
n = 6
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
ctx = TreeAttention(n_layers=n, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
ctx.restore(*snap)
for layer in range(n):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c:
            ctx.write_kv(layer, int(node), (torch.rand((c, hkv, d), device="cuda") * 2 - 1).bfloat16(),
                         (torch.rand((c, hkv, d), device="cuda") * 2 - 1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((n, L, hq, d), device="cuda") * 2 - 1).bfloat16()
out = torch.empty_like(q)
ctx.prepare(128)
for _ in range(3):
    for layer in range(n):
        ctx.attend(layer, q[layer], out[layer])
torch.cuda.synchronize()
tls = []
for layer in range(n):
    tl = torch.tensor([2**63 - 1, 0] * 5, dtype=torch.int64, device="cuda")
    tls.append(tl)
ctx.prepare(128)
torch.cuda.synchronize()
for layer in range(n):
    ctx.set_option("timeline_ptr", tls[layer].data_ptr())
    ctx.attend(layer, q[layer], out[layer])
torch.cuda.synchronize()
t0 = int(tls[0][0])
print(f"{name}: per layer (us rel. to layer 0 attention start): attn start/end, merge start/end, "
      "CTA entry first/last, staged first/last")
for layer in range(n):
    a = [int(x) for x in tls[layer].cpu()]
    ms = "-" if a[2] > 2**62 else f"{(a[2] - t0) / 1e3:8.2f} {(a[3] - t0) / 1e3:8.2f}"
    ex = "" if a[4] > 2**62 else " ".join(f"{(x - t0) / 1e3:8.2f}" for x in a[4:8])
    if a[8] < 2**62:
        ex += "   merge entry " + " ".join(f"{(x - t0) / 1e3:8.2f}" for x in a[8:10])
    print(f"  {layer}: {(a[0] - t0) / 1e3:8.2f} {(a[1] - t0) / 1e3:8.2f}   {ms}   {ex}   dur {(a[1] - a[0]) / 1e3:.2f}")
