"""CTA phase timeline of one attention launch (debug): start, items done
(bulk copies landed), end (after the fused merge), from the TRACE
instantiation's globaltimer marks.

    python scripts/trace_phases.py [config] [option=value ...]"""
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
NL = 4 if cfg["n_layers"] >= 4 else cfg["n_layers"]
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
res = []
for rep in range(6):
    for layer in range(NL):
        tr.zero_()
        ctx.attend(layer, q)   # isolated launches: this one alone on the GPU
        torch.cuda.synchronize()
        t = tr.cpu().numpy().reshape(n_cta, 256)
        t0 = t[:, 0].min()
        res.append(((t[:, 0] - t0) / 1e3, (t[:, 6] - t0) / 1e3, (t[:, 1] - t0) / 1e3, np.where(t[:, 7] > 0, (t[:, 7] - t0) / 1e3, np.nan), np.where(t[:, 236] > 0, (t[:, 236] - t0) / 1e3, np.nan), np.where(t[:, 237] > 0, (t[:, 237] - t0) / 1e3, np.nan), np.where(t[:, 200:211] > 0, (t[:, 200:211] - t0) / 1e3, np.nan), np.where(t[:, 238] > 0, (t[:, 238] - t0) / 1e3, np.nan), np.where(t[:, 239] > 0, (t[:, 239] - t0) / 1e3, np.nan)))
st, it, en, wd, md, pu, fw, fe, pf = (np.stack([r[i] for r in res[NL:]]) for i in range(9))
pc = lambda a: " ".join(f"{x:6.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
print(f"{name} {' '.join(opts)}: {n_cta} CTAs, {len(res) - NL} isolated launches; percentiles 0/10/50/90/100 (us from first CTA start)")
print("  CTA start     ", pc(st))
print("  items done    ", pc(it))
print("  CTA end       ", pc(en))
print("  merge phase   ", pc(en - it))
print("  span (max end) mean %.2f" % en.max(axis=1).mean())
pn = lambda a: " ".join(f"{x:6.2f}" for x in np.nanpercentile(a, [0, 10, 50, 90, 100]))
last = it.max(axis=1, keepdims=True)
print("  waits done - last items done  ", pn(wd - last))
print("  merge loop end - last items   ", pn(md - last))
print("  CTA end - last items done     ", pn(en - last))
print("  publish - own items done      ", pn(pu - it))
print("  pre-fence - own items done    ", pn(pf - it))
print("  pre-fence (abs)               ", pn(pf))
lastpf = np.nanmax(pf, axis=1, keepdims=True)
print("  CTA end - last pre-fence      ", pn(en - lastpf))
print("  first wait - last pre-fence   ", pn(fw - lastpf[..., None]))
print("  fence done - pre-fence        ", pn(fe - pf))
print("  publish - last items done     ", pn(pu - last))
print("  first wait done - last items  ", pn(fw - last[..., None]))
print("  first wait done - own publish ", pn(fw - pu[..., None]))
