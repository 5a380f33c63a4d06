import os, sys
sys.path.insert(0, '/root/repo'); os.chdir(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import numpy as np, torch, bench
from paper_2404_00242_b200 import TreeAttention
name = sys.argv[1] if len(sys.argv) > 1 else "few_shot"
cfg = dict(bench.CONFIGS[name]); snap = bench.build_snapshot(cfg); root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]; n_loc = cfg.get("n_local_kv_heads") or hkv
NL = 2
ctx = TreeAttention(n_layers=NL, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16, n_local_kv_heads=n_loc)
ctx.restore(*snap)
for layer in range(NL):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c: ctx.write_kv(layer, int(node), (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16(), (torch.rand((c, n_loc, d), device="cuda") * 2 - 1).bfloat16())
L = len(ctx.leaves()); q = (torch.rand((L, ctx.n_local_q_heads, d), device="cuda") * 2 - 1).bfloat16()
ctx.prepare(128); S = ctx.schedule(128); n_cta = S["n_ctas"]
NB = 8
trs = [torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda") for _ in range(NB)]; outs = [torch.empty_like(q) for _ in range(NB)]
D = []
for rep in range(5):
    for t_ in trs: t_.zero_()
    torch.cuda.synchronize()
    for i in range(NB):
        ctx.set_option("trace_ptr", trs[i].data_ptr()); ctx.attend(i % NL, q, outs[i])
    torch.cuda.synchronize()
    if rep:
        for t_ in trs[1:]:
            t = t_.cpu().numpy().reshape(n_cta, 256); D.append((t[:, 6] - np.maximum(t[:, 0], t[:, 40])) / 1e3)
dm = np.median(np.array(D), axis=0)
it, cb = S["items"], S["cta_begin"]
# lane id of each item = items[:,6]; lanes with the same (head, tile range start) ... print per CTA
from collections import defaultdict
by = defaultdict(list)
for c in range(n_cta):
    its = list(range(int(cb[c]), int(cb[c + 1])))
    if not its: continue
    key = tuple((int(it[i][6]), int(it[i][4]) * ctx.group) for i in its)
    lanes = [int(it[i][6]) for i in its]; rows = [int(it[i][4]) * ctx.group for i in its]; nt = sum(int(it[i][2] - it[i][1]) for i in its)
    kind = "+".join(("L%d:%dr" % (l, r)) for l, r in zip(lanes, rows))
    by[(len(its), nt, tuple(sorted(set(lanes))) if len(set(lanes)) < 3 else "many")].append(dm[c])
for k in sorted(by, key=lambda k: str(k)):
    v = by[k]; print(k, len(v), round(float(np.mean(v)), 2))
