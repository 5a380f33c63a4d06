"""Per-tile pipeline trace of the MMA kernel's CTA (0,0) on the few-shot config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_00242_b200 import TreeAttention
cfg = dict(bench.CONFIGS["few_shot"]); cfg["n_layers"] = 2
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
ctx = TreeAttention(n_layers=2, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c)+15)//16 for c in cnt))+16)
for kv in sys.argv[1:]:
    k, v = kv.split("="); ctx.set_option(k, int(v))
ctx.restore(*snap)
for layer in range(2):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c: ctx.write_kv(layer, int(node), (torch.rand((c, 8, 128), device="cuda")*2-1).bfloat16(), (torch.rand((c, 8, 128), device="cuda")*2-1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((L, 32, 128), device="cuda")*2-1).bfloat16()
tr = torch.zeros(512 + 4*4096, dtype=torch.int64, device="cuda")
ctx.set_option("trace_ptr", tr.data_ptr())
ctx.prepare(128)
for layer in (0, 1, 0):
    ctx.attend(layer, q)
torch.cuda.synchronize()
full = tr.cpu().numpy()
t = full[:512].reshape(64, 8)
base = t[0, 0]
names = ["prod_issue", "qk_data", "qk_issued", "sm_S_seen", "sm_P_pub", "pv_issued", "stage_free"]
print("cycles rel. to first producer issue; per tile:")
print("tile " + " ".join(f"{n:>11s}" for n in names))
for i in range(64):
    if t[i].any():
        print(f"{i:4d} " + " ".join(f"{(x - base) if x else 0:11d}" for x in t[i, :7]))

c = full[512:].reshape(4096, 4)
c = c[c[:, 1] > 0]
t0 = c[:, 0].min()
dur = (c[:, 1] - c[:, 0]) / 1000.0
print(f"CTAs {len(c)}  kernel span {(c[:,1].max()-t0)/1000:.1f} us  cta dur mean {dur.mean():.1f} max {dur.max():.1f} us")
order = np.argsort(-dur)
print("slowest CTAs: start(us) dur(us) sm groups rows")
for i in order[:12]:
    print(f"  {(c[i,0]-t0)/1000:7.1f} {dur[i]:7.1f} {c[i,2]:4d} {c[i,3]>>32:5d} {c[i,3]&0xffffffff:5d}")
print("dur by rows (live rows -> mean us, mean us per tile):")
rows = c[:, 3] & 0xffffffff
grp = c[:, 3] >> 32
for r in sorted(set(rows.tolist())):
    m = rows == r
    print(f"  rows {r:4d}: n={m.sum():4d} dur {dur[m].mean():6.1f} us, per tile {(dur[m] / np.maximum(1, (grp[m]+7)//8)).mean():5.2f} us")
