"""Item switches in the tcgen05 kernel's pipeline trace (TRACE build path,
selected by trace_ptr): for CTAs running several items, the gap between the
last tile of item k (P published, epilogue) and the first tile of item k+1
(K issued, S seen, P published), against the within-item tile period.
    python scripts/trace_items.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_00242_b200 import TreeAttention

NT = 20
name = sys.argv[1] if len(sys.argv) > 1 else "reasoning"
cfg = dict(bench.CONFIGS[name])
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
n_loc = cfg.get("n_local_kv_heads") or hkv
ctx = TreeAttention(n_layers=2, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16, n_local_kv_heads=n_loc)
ctx.restore(*snap)
for layer in range(2):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c:
            ctx.write_kv(layer, int(node), (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16(),
                         (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((L, ctx.n_local_q_heads, d), device="cuda") * 2 - 1).bfloat16()
ctx.prepare(128)
for layer in (0, 1, 0, 1):
    ctx.attend(layer, q)
torch.cuda.synchronize()
S = ctx.schedule(128)
n_cta = S["n_ctas"]
tr = torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda")
ctx.set_option("trace_ptr", tr.data_ptr())
ctx.attend(1, q)
torch.cuda.synchronize()
ctx.set_option("trace_ptr", 0)
t = tr.cpu().numpy().reshape(n_cta, 256)
it, cb = S["items"], S["cta_begin"]
within, switch = [], []
shown = 0
for c in range(n_cta):
    items = list(range(int(cb[c]), int(cb[c + 1])))
    nt = min(int(t[c, 3]), NT)
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8).astype(np.int64)
    bounds = np.cumsum([int(it[i][2] - it[i][1]) for i in items])[:-1]
    for i in range(1, nt):
        gap = ev[i, 1] - ev[i - 1, 6]          # P(i-1) published -> S(i) seen
        per = ev[i, 6] - ev[i - 1, 6]          # P period
        (switch if i in bounds else within).append((gap, per, ev[i, 1] - ev[i, 0], ev[i, 6] - ev[i, 1]))
    if len(items) >= 3 and shown < 3 and nt >= bounds[-1] + 1:
        shown += 1
        b = ev[0, 0]
        print(f"CTA {c}: items (rows, tiles) {[(int(it[i][4]) * ctx.group, int(it[i][2] - it[i][1])) for i in items]}")
        print("   tile  K_issued    S_seen  S_masked  max_xchg  V_issue  rescaled     P_pub   epi(k)")
        for i in range(nt):
            mark = " <- item start" if i in bounds else ""
            print("   %4d" % i + "".join(" %9d" % ((x - b) if x else -1) for x in ev[i]) + mark)
# per-item marks (slots 198 + 6k + j) relative to the previous item's last P
print("item switch phases (clk after item k's last P): item k: epi O_FULL, staging free, copies issued | item k+1: softmax setup done, at S wait, QK past Q_FULL, QK(first) committed, S seen, PV(first) committed")
sw = []
for c in range(n_cta):
    items = list(range(int(cb[c]), int(cb[c + 1])))
    nt = min(int(t[c, 3]), NT)
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8).astype(np.int64)
    ends = np.cumsum([int(it[i][2] - it[i][1]) for i in items])
    for k in range(min(len(items) - 1, 2)):
        last = ends[k] - 1
        if last + 1 >= nt:
            break
        p = ev[last, 6]
        m = t[c, 198 + 8 * k: 206 + 8 * k].astype(np.int64)
        n = t[c, 198 + 8 * (k + 1): 206 + 8 * (k + 1)].astype(np.int64)
        sw.append([m[2] - p, m[3] - p, m[4] - p, n[6] - p, n[7] - p, n[0] - p, n[1] - p, ev[last + 1, 1] - p, n[5] - p])
if sw:
    sw = np.array(sw)
    print("  median:", " ".join(f"{x:8.0f}" for x in np.median(sw, 0)), f"  (n={len(sw)})")
    print("  p90   :", " ".join(f"{x:8.0f}" for x in np.percentile(sw, 90, axis=0)))
w, s = np.array(within), np.array(switch)
hdr = "P(t-1)->S(t) gap, P period, K issue->S seen, S seen->P"
if len(w):
    print(f"{name} within items (n={len(w)}): {hdr}:", " ".join(f"{x:8.0f}" for x in np.median(w, 0)))
if len(s):
    print(f"{name} item switches (n={len(s)}): {hdr}:", " ".join(f"{x:8.0f}" for x in np.median(s, 0)))
