"""Fit the schedule cost model to measured CTA durations (debug / tuning).

Runs the pipeline trace on a config and regresses each CTA's duration on its
box rows, tiles, items and attended pairs; prints the fitted coefficients in
the units of the cost model (box rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_00242_b200 import TreeAttention

names = sys.argv[1:] or ["few_shot"]
X, Y = [], []
for name in names:
    cfg = dict(bench.CONFIGS[name])
    snap = bench.build_snapshot(cfg)
    root, ids, par, cnt = snap
    hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
    ctx = TreeAttention(n_layers=2, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                        max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16)
    ctx.restore(*snap)
    for layer in range(2):
        for node, c in zip(ids, cnt):
            c = int(c)
            if c:
                ctx.write_kv(layer, int(node), (torch.rand((c, hkv, d), device="cuda") * 2 - 1).bfloat16(),
                             (torch.rand((c, hkv, d), device="cuda") * 2 - 1).bfloat16())
    L = len(ctx.leaves())
    q = (torch.rand((L, hq, d), device="cuda") * 2 - 1).bfloat16()
    ctx.prepare(128)
    for layer in (0, 1, 0, 1):
        ctx.attend(layer, q)
    S = ctx.schedule(128)
    G = ctx.group
    for rep in range(3):
        tr = torch.zeros(S["n_ctas"] * 256, dtype=torch.int64, device="cuda")
        ctx.set_option("trace_ptr", tr.data_ptr())
        ctx.attend(rep % 2, q)
        torch.cuda.synchronize()
        ctx.set_option("trace_ptr", 0)
        t = tr.cpu().numpy().reshape(S["n_ctas"], 256)
        dur = (t[:, 1] - t[:, 0]) / 1e3
        for c in range(S["n_ctas"]):
            rows = tiles = items = pairs = 0
            for i in range(S["cta_begin"][c], S["cta_begin"][c + 1]):
                items += 1
                tb, te = int(S["items"][i][1]), int(S["items"][i][2])
                for tt in range(tb, te):
                    tiles += 1
                    ng = int(S["tile_ng"][tt])
                    rows += 16 * ng
                    g0 = int(S["tile_grp_begin"][tt])
                    for g in range(g0, g0 + ng):
                        info = int(S["grp_info"][g])
                        pairs += (info & 0xFF) * ((info >> 20) - ((info >> 8) & 0xFFF)) * G
            if items:
                X.append([rows, tiles, items, pairs / 16384.0, 1.0])
                Y.append(dur[c])
X, Y = np.array(X), np.array(Y)
coef, res, *_ = np.linalg.lstsq(X, Y, rcond=None)
pred = X @ coef
print("fit: us = %.4f*box_rows + %.3f*tiles + %.3f*items + %.3f*dense_tiles + %.3f" % tuple(coef))
print("in box-row units: tile_cost %.1f  item_cost %.1f  row_cost %.1f  (const %.1f)" %
      (coef[1] / coef[0], coef[2] / coef[0], coef[3] / coef[0], coef[4] / coef[0]))
print("residual rms %.2f us, duration mean %.2f max %.2f" % (np.sqrt(np.mean((pred - Y) ** 2)), Y.mean(), Y.max()))
