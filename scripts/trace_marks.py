"""Phase marks of the tcgen05 attention launch (debug): per CTA globaltimer at
entry, staged, first K issued, first / last P, epilogue start, last copy
issued, copies landed, published, merge waits done, end (slots 180..191 of
the TRACE instantiation), over isolated launches.

    python scripts/trace_marks.py [config] [option=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_00242_b200 import TreeAttention

name = sys.argv[1] if len(sys.argv) > 1 and "=" not in sys.argv[1] else "few_shot"
opts = [a for a in sys.argv[1:] if "=" in a]
cfg = dict(bench.CONFIGS[name])
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
NL = 4
n_loc = cfg.get("n_local_kv_heads") or hkv
ctx = TreeAttention(n_layers=NL, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16, n_local_kv_heads=n_loc)
for kv in opts:
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
ctx.restore(*snap)
for layer in range(NL):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c:
            ctx.write_kv(layer, int(node), (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16(),
                         (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((L, ctx.n_local_q_heads, d), device="cuda") * 2 - 1).bfloat16()
ctx.prepare(128)
S = ctx.schedule(128)
n_cta = S["n_ctas"]
tr = torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda")
ctx.set_option("trace_ptr", tr.data_ptr())
names = ["entry", "staged", "-", "first K", "first P", "last P", "epi start", "last copy", "copies done",
         "published", "waits done", "end", "barrier", "fenced"]
rows = []
for rep in range(6):
    for layer in range(NL):
        tr.zero_()
        ctx.attend(layer, q)
        torch.cuda.synchronize()
        T = tr.cpu().numpy().reshape(n_cta, 256)
        g0, c0, g1, c1 = (T[:, 192 + i].astype(np.float64) for i in range(4))
        f = (c1 - c0) / np.maximum(g1 - g0, 1)   # SM clocks per ns
        t = np.concatenate([T[:, 180:192], T[:, 196:198]], axis=1).astype(np.float64)
        t[t == 0] = np.nan
        t = g0[:, None] + (t - c0[:, None]) / f[:, None]
        if rep >= 1:
            rows.append((t - np.nanmin(t[:, 0])) / 1e3)
A = np.stack(rows)   # launches x CTAs x marks
print(f"{name} {' '.join(opts)}: {n_cta} CTAs, {A.shape[0]} isolated launches; us from the first CTA entry")
print("  mark            p0     p10    p50    p90    p100   (over CTAs and launches)")
for i, nm in enumerate(names):
    if nm == "-" or np.all(np.isnan(A[:, :, i])):
        continue
    print(f"  {nm:12s} " + " ".join(f"{x:6.2f}" for x in np.nanpercentile(A[:, :, i], [0, 10, 50, 90, 100])))
end = np.nanmax(A[:, :, 11], axis=1)
print(f"  launch span mean {end.mean():.2f}")
# the critical CTA of each launch: the one that ends last; its phase durations
crit = np.nanargmax(A[:, :, 11], axis=1)
C = A[np.arange(A.shape[0]), crit]
print("  critical CTA phases (median over launches):")
for i, nm in enumerate(names):
    if nm != "-":
        print(f"    {nm:12s} {np.nanmedian(C[:, i]):6.2f}")
# last copies landed over all CTAs vs end
lastcopy = np.nanmax(A[:, :, 8], axis=1)
print(f"  last 'copies done' over CTAs: median {np.median(lastcopy):.2f}; end - that: median {np.median(end - lastcopy):.2f}")
