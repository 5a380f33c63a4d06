"""Is CTA imbalance systematic or random?  Light-trace build
(-DTA_LIGHT_TRACE=1), NB back-to-back launches of one config: per CTA the
time from its launch's first entry to its last P (slot 4) and last epilogue
copy (slot 5), its SM (slot 41) and its modelled cost.  Prints the spread,
the correlation of a CTA's lateness across launches (same blockIdx), across
launches on the same SM, and with the modelled cost.
    python scripts/cta_variance.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_00242_b200 import TreeAttention

name = sys.argv[1] if len(sys.argv) > 1 else "few_shot"
cfg = dict(bench.CONFIGS[name])
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
NL = 4
n_loc = cfg.get("n_local_kv_heads") or hkv
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
n_cta = S["n_ctas"]
NB, REPS = 8, 6
trs = [torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda") for _ in range(NB)]
outs = [torch.empty_like(q) for _ in range(NB)]
LP, LC, SM = [], [], []
for rep in range(REPS):
    for t_ in trs:
        t_.zero_()
    torch.cuda.synchronize()
    for i in range(NB):
        ctx.set_option("trace_ptr", trs[i].data_ptr())
        ctx.attend(i % NL, q, outs[i])
    torch.cuda.synchronize()
    if rep == 0:
        continue
    for t_ in trs[1:]:   # launch 0 has no predecessor
        t = t_.cpu().numpy().reshape(n_cta, 256)
        t0 = t[:, 0].min()
        LP.append((t[:, 4] - t0) / 1e3)
        LC.append((t[:, 5] - t0) / 1e3)
        SM.append(t[:, 41])
LP, LC, SM = np.array(LP), np.array(LC), np.array(SM)
# modelled cost per CTA: tiles' box rows (the host model's KV term) + items
it = S["items"]
cb = S["cta_begin"]
pc = lambda a: " ".join(f"{x:6.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
print(f"{name}: {n_cta} CTAs, {LP.shape[0]} launches")
print("last P (us from launch's first entry)   p0 p10 p50 p90 p100:", pc(LP))
print("last copy                                                  :", pc(LC))
spread = LC.max(axis=1) - np.median(LC, axis=1)
print("per launch: max - median last copy", pc(spread))
# lateness = deviation from the launch median
dev = LC - np.median(LC, axis=1, keepdims=True)
m_cta = dev.mean(axis=0)
resid = dev - m_cta
print(f"lateness variance: total {dev.var():.3f}, explained by blockIdx (systematic) {m_cta.var():.3f}, residual {resid.var():.3f}")
# same SM across launches
sm_dev = {}
for r in range(dev.shape[0]):
    for c in range(n_cta):
        sm_dev.setdefault(int(SM[r, c]), []).append(dev[r, c] - m_cta[c])
sm_m = np.array([np.mean(v) for v in sm_dev.values()])
print(f"after blockIdx: variance explained by SM {sm_m.var():.3f} of {resid.var():.3f}; blockIdx->SM stable: "
      f"{np.mean([np.all(SM[:, c] == SM[0, c]) for c in range(n_cta)]):.2f}")
order = np.argsort(-m_cta)
print("latest CTAs (mean lateness us, SM of launch 0, items):",
      [(int(c), round(float(m_cta[c]), 2), int(SM[0, c]), int(cb[c + 1] - cb[c])) for c in order[:10]])
print("earliest CTAs:", [(int(c), round(float(m_cta[c]), 2), int(SM[0, c]), int(cb[c + 1] - cb[c])) for c in order[-6:]])
# lateness vs SM die (SM id parity / halves)
smh = SM < 74
print(f"mean lateness SM<74 {dev[smh].mean():.3f}, SM>=74 {dev[~smh].mean():.3f}; even SM {dev[SM % 2 == 0].mean():.3f}, odd {dev[SM % 2 == 1].mean():.3f}")
# modelled KV rows per CTA (sum of its tiles' box rows) and item count
nrows = np.zeros(n_cta)
ntile = np.zeros(n_cta)
boxes = S["tile_boxes"]
rows_t = np.array([sum(16 << (int(b) & 3) for b in boxes[t][:int(S["tile_nbox"][t])]) for t in range(len(boxes))]) if len(boxes) else np.zeros(0)
for c in range(n_cta):
    for i in range(int(cb[c]), int(cb[c + 1])):
        nrows[c] += rows_t[int(it[i, 1]):int(it[i, 2])].sum()
        ntile[c] += int(it[i, 2]) - int(it[i, 1])
for nm, x in (("box rows", nrows), ("tiles", ntile), ("items", np.diff(cb))):
    if x.std() > 0:
        print(f"corr(mean lateness, {nm}) = {np.corrcoef(m_cta, x)[0, 1]:.3f}   ({nm}: {pc(x)})")
np.savez(f"gpurun_out/cta_variance_{name}.npz", LP=LP, LC=LC, SM=SM)
