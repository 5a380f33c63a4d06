"""CTA spans of the PRODUCT kernel (each mark is a %globaltimer read, which
itself takes a fraction of a microsecond: consecutive marks with nothing
between them read ~0.5 us apart, so use differences between distant marks) (built with -DTA_LIGHT_TRACE=1, see
scripts/build_variant.sh): entry, items done, exit per CTA (globaltimer), over
isolated launches.   python scripts/light_spans.py [config] [option=value ...]"""
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
B2B = os.environ.get("B2B")
if B2B:
    # back-to-back launches (as in the bench's graph): one trace buffer per launch
    NB = 8
    trs = [torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda") for _ in range(NB)]
    outs = [torch.empty_like(q) for _ in range(NB)]
    for rep in range(3):
        for t_ in trs:
            t_.zero_()
        torch.cuda.synchronize()
        for i in range(NB):
            ctx.set_option("trace_ptr", trs[i].data_ptr())
            ctx.attend(i % NL, q, outs[i])
        torch.cuda.synchronize()
    T = [t_.cpu().numpy().reshape(n_cta, 256) for t_ in trs]
    g0 = min(t[:, 0].min() for t in T)
    print(f"{name} back-to-back: per launch (us from launch 0's first entry): first entry, last entry, median items done, last exit")
    for i, t in enumerate(T):
        print(f"  {i}: {(t[:, 0].min() - g0) / 1e3:8.2f} {(t[:, 0].max() - g0) / 1e3:8.2f} {(np.median(t[:, 6]) - g0) / 1e3:8.2f} {(t[:, 1].max() - g0) / 1e3:8.2f}"
              f"   first K issue med {(np.median(t[:, 2]) - g0) / 1e3:8.2f}  last P med {(np.median(t[:, 4]) - g0) / 1e3:8.2f}  last copy med/max {(np.median(t[:, 5]) - g0) / 1e3:8.2f} {(t[:, 5].max() - g0) / 1e3:8.2f}")
    # merge phase of launch 3: per CTA publish, last wait done, last merge done, exit
    t = T[3]
    t0 = t[:, 0].min()
    pub = np.where(t[:, 9] > 0, (t[:, 9] - t0) / 1e3, np.nan)
    wd = np.where(t[:, 12:23] > 0, (t[:, 12:23] - t0) / 1e3, np.nan)
    md = np.where(t[:, 24:35] > 0, (t[:, 24:35] - t0) / 1e3, np.nan)
    ex = (t[:, 1] - t0) / 1e3
    lc = (t[:, 5] - t0) / 1e3
    pc = lambda a: " ".join(f"{x:6.2f}" for x in np.nanpercentile(a, [0, 10, 50, 90, 100]))
    print("launch 3 merge phase (us from its first entry): p0 p10 p50 p90 p100 over CTAs")
    print("  last copy      ", pc(lc[lc > 0]))
    print("  copies landed  ", pc(np.where(t[:, 35] > 0, (t[:, 35] - t0) / 1e3, np.nan)))
    print("  CTA barrier    ", pc(np.where(t[:, 36] > 0, (t[:, 36] - t0) / 1e3, np.nan)))
    print("  fenced         ", pc(np.where(t[:, 37] > 0, (t[:, 37] - t0) / 1e3, np.nan)))
    print("  published      ", pc(pub))
    print("  last wait done ", pc(np.nanmax(wd, axis=1)))
    print("  first wait done", pc(np.nanmin(wd, axis=1)))
    print("  last merge done", pc(np.nanmax(md, axis=1)))
    print("  exit           ", pc(ex))
    print("  merge rows per warp: max wait->merge done", pc(np.nanmax(md - wd, axis=1)))
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = []
ev = []
for rep in range(8):
    for layer in range(NL):
        tr.zero_()
        torch.cuda.synchronize()
        e0.record()
        ctx.attend(layer, q)
        e1.record()
        torch.cuda.synchronize()
        t = tr.cpu().numpy().reshape(n_cta, 256)
        if rep:
            t0 = t[:, 0].min()
            R.append(np.stack([(t[:, i] - t0) / 1e3 if i != 9 else t[:, 9] for i in (0, 6, 1, 2, 3, 7, 4, 5, 38, 39, 40)], axis=1))
            ev.append(e0.elapsed_time(e1) * 1e3)
R = np.stack(R)
pc = lambda a: " ".join(f"{x:6.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
print(f"{name} {' '.join(opts)}: {n_cta} CTAs, {R.shape[0]} isolated launches, event time median {np.median(ev):.2f} us")
print("                 p0     p10    p50    p90    p100  (us from the first CTA entry)")
print("  entry        ", pc(R[:, :, 0]))
print("  items done   ", pc(R[:, :, 1]))
print("  exit         ", pc(R[:, :, 2]))
print("  items span   ", pc(R[:, :, 1] - R[:, :, 0]))
print("  exit - items ", pc(R[:, :, 2] - R[:, :, 1]))
print("  last exit    ", pc(R[:, :, 2].max(axis=1)))
print("  exit - last items done", pc(R[:, :, 2] - R[:, :, 1].max(axis=1, keepdims=True)))
nt = np.array([S["cta_tiles"][c] for c in range(n_cta)]) if "cta_tiles" in S else None
ok = ~np.isnan(R[:, :, 3]) & (R[:, :, 3] > -1e5)
for nm, i in (("TMEM + barriers", 8), ("head landed", 9), ("after pdl wait", 10), ("first K issue", 3), ("first P", 4), ("P tile 4", 5), ("last P", 6), ("last copy issued", 7)):
    v = R[:, :, i]
    v = v[(v > -1e5) & (v < 1e5)]
    print(f"  {nm:16s}", pc(v))
rate = (R[:, :, 6] - R[:, :, 5])
print("  last P - P4      ", pc(rate[(rate > 0) & (rate < 1e5)]))
print("  exit - last copy ", pc((R[:, :, 2] - R[:, :, 7])[(R[:, :, 7] > 0) & (R[:, :, 7] < 1e5)]))
print("  last copy - last P", pc((R[:, :, 7] - R[:, :, 6])[(R[:, :, 7] > 0) & (R[:, :, 7] < 1e5)]))
