"""Fit the schedule cost model (host.cpp step 3) to the PRODUCT kernel's
per-CTA durations.  Light-trace build (-DTA_LIGHT_TRACE=1, see
scripts/build_variant.sh), NB back-to-back launches per config as in the
bench's graph; a CTA's duration = its items-done mark (slot 6, after its
epilogue copies landed) - the later of its entry (slot 0) and the end of
its dependency wait (slot 40: the previous launch has finished).  Regresses durations on box
rows, tiles, items and dense-tile softmax work; prints the coefficients in
box-row units (tile_cost, item_cost, row_cost) and how well the current and
the fitted constants predict.   python scripts/calibrate2.py cfg [cfg ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_00242_b200 import TreeAttention


def features(S, G):
    it, cb = S["items"], S["cta_begin"]
    out = []
    for c in range(S["n_ctas"]):
        rows = tiles = items = pairs = boxes = 0
        for i in range(int(cb[c]), int(cb[c + 1])):
            items += 1
            for tt in range(int(it[i][1]), int(it[i][2])):
                tiles += 1
                boxes += int(S["tile_nbox"][tt])
                ng = int(S["tile_ng"][tt])
                rows += 16 * ng
                g0 = int(S["tile_grp_begin"][tt])
                for g in range(g0, g0 + ng):
                    info = int(S["grp_info"][g])
                    pairs += (info & 0xFF) * ((info >> 20) - ((info >> 8) & 0xFFF)) * G
        out.append([rows, tiles, boxes, items, pairs / 16384.0])
    return np.array(out, dtype=np.float64)


X, Y, TAG = [], [], []
for name in sys.argv[1:] or ["few_shot"]:
    cfg = dict(bench.CONFIGS[name])
    snap = bench.build_snapshot(cfg)
    root, ids, par, cnt = snap
    hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
    n_loc = cfg.get("n_local_kv_heads") or hkv
    NL = 2
    ctx = TreeAttention(n_layers=NL, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                        max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16, n_local_kv_heads=n_loc)
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
    F = features(S, ctx.group)
    n_cta = S["n_ctas"]
    NB = 8
    trs = [torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda") for _ in range(NB)]
    outs = [torch.empty_like(q) for _ in range(NB)]
    D = []
    for rep in range(5):
        for t_ in trs:
            t_.zero_()
        torch.cuda.synchronize()
        for i in range(NB):
            ctx.set_option("trace_ptr", trs[i].data_ptr())
            ctx.attend(i % NL, q, outs[i])
        torch.cuda.synchronize()
        if rep:
            for t_ in trs[1:]:
                t = t_.cpu().numpy().reshape(n_cta, 256)
                D.append((t[:, 6] - np.maximum(t[:, 0], t[:, 40])) / 1e3)
    ctx.set_option("trace_ptr", 0)
    D = np.array(D)
    dm = np.median(D, axis=0)
    has = F[:, 2] > 0
    print(f"{name}: {n_cta} CTAs, {has.sum()} with items; duration p0/p50/p100 {dm[has].min():.2f} {np.median(dm[has]):.2f} {dm[has].max():.2f} us"
          f"; systematic sd {dm[has].std():.2f}, launch-to-launch sd {np.mean(D[:, has].std(axis=0)):.2f}")
    X.append(F[has])
    Y.append(dm[has])
    TAG += [name] * int(has.sum())
X = np.concatenate(X)
Y = np.concatenate(Y)
TAG = np.array(TAG)
A = np.concatenate([X, np.ones((len(X), 1))], axis=1)
coef, *_ = np.linalg.lstsq(A, Y, rcond=None)
print("fit: us = %.5f*box_rows + %.4f*tiles + %.4f*boxes + %.3f*items + %.4f*dense_tiles + %.3f" % tuple(coef))
print("in box-row units: tile_cost %.1f  box_cost %.1f  item_cost %.1f  row_cost %.1f  (const %.1f)" %
      tuple(coef[1:] / coef[0]))
cur = X @ np.array([1.0, 24.0, 0.0, 300.0, 15.0])
for name in dict.fromkeys(TAG):
    m = TAG == name
    pf = A[m] @ coef
    # how well each model ranks this config's CTAs (a partition only needs relative costs)
    r_cur = np.corrcoef(cur[m], Y[m])[0, 1] if cur[m].std() > 0 else float("nan")
    r_fit = np.corrcoef(pf, Y[m])[0, 1] if pf.std() > 0 else float("nan")
    print(f"  {name:20s} corr(current model, dur) {r_cur:.3f}  corr(fit, dur) {r_fit:.3f}  fit rms {np.sqrt(np.mean((pf - Y[m]) ** 2)):.2f} us")
np.savez("gpurun_out/calibrate2.npz", X=X, Y=Y, TAG=TAG)
fit = {k: max(0, int(round(v))) for k, v in zip(("tile_cost", "box_cost", "item_cost", "row_cost"), coef[1:5] / coef[0])}
print("opts:", " ".join(f"--opt {k}={v}" for k, v in fit.items()))
with open("gpurun_out/calibrate2_opts.txt", "w") as f:
    f.write(" ".join(f"--opt {k}={v}" for k, v in fit.items()))
