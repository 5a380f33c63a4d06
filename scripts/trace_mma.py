"""Pipeline trace of the persistent tcgen05 kernel on a bench config (debug).

    python scripts/trace_mma.py [config] [option=value ...]

Prints per-CTA durations (globaltimer) and per-tile pipeline events (clock64)
of a few CTAs (see the TRACE comment in csrc/attn_mma.cu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench

NT = 20   # traced tiles per CTA (TRACE_TILES in csrc/attn_mma.cu)
from paper_2404_00242_b200 import TreeAttention

name = sys.argv[1] if len(sys.argv) > 1 and "=" not in sys.argv[1] else "few_shot"
opts = [a for a in sys.argv[1:] if "=" in a]
cfg = dict(bench.CONFIGS[name])
cfg["n_layers"] = 2
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
hkv, hq, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
ctx = TreeAttention(n_layers=2, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16", out_dtype="bf16",
                    max_pages=int(sum((int(c) + 15) // 16 for c in cnt)) + 16)
for kv in opts:
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
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
torch.cuda.synchronize()
S = ctx.schedule(128)
n_cta = S["n_ctas"]
tr = torch.zeros(n_cta * 256, dtype=torch.int64, device="cuda")
ctx.set_option("trace_ptr", tr.data_ptr())
ctx.prepare(128)
ctx.attend(1, q)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(n_cta, 256)
t0 = t[:, 0].min()
start = (t[:, 0] - t0) / 1e3
end = (t[:, 1] - t0) / 1e3
dur = end - start
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/dur_{name}.npy", np.stack([start, end]))
print(f"{name}: CTAs {n_cta}, kernel span {end.max():.2f} us, start spread {start.max():.2f} us, "
      f"dur min/mean/max {dur.min():.2f}/{dur.mean():.2f}/{dur.max():.2f} us")
for c in list(np.argsort(-dur)[:3]) + list(np.argsort(dur)[:2]):
    nt = int(t[c, 3])
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8)
    b = ev[0, 0]
    its = [i for i in range(S["cta_begin"][c], S["cta_begin"][c + 1])]
    desc = [(int(S["items"][i][0]), int(S["items"][i][2] - S["items"][i][1]), int(S["items"][i][4]) * ctx.group)
            for i in its]
    print(f"CTA {c} sm {t[c,2]} start {start[c]:.2f} dur {dur[c]:.2f} us tiles {nt} items(head,tiles,rows) {desc}")
    print("   tile  K_issued    S_seen  S_masked  max_xchg  O_full-1  rescaled     P_pub       epi  (clk rel. first K issue)")
    for i in range(min(nt, NT)):
        print("   %4d" % i + "".join(" %9d" % ((x - b) if x else -1) for x in ev[i]))
    for nm, sl in (("first", 240), ("last", 248)):
        epi = t[c, sl:sl + 4]
        print(f"   {nm} item epilogue: O_full_seen  l_xchg_start  O_loaded  stored:",
              " ".join(str((x - b) if x else -1) for x in epi))

# phase averages per tile over all CTAs, grouped by the CTA's first item rows
print("\nper-tile phase means (clk): rows  n_cta  tile_period  S_wait  pass1  xchg  O_wait  rescale  pass2")
groups = {}
for c in range(n_cta):
    nt = min(int(t[c, 3]), NT)
    if nt < 3:
        continue
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8)[:nt].astype(np.float64)
    i0 = S["cta_begin"][c]
    rows = int(S["items"][i0][4]) * ctx.group
    period = np.diff(ev[:, 1]).mean()
    ph = [(ev[1:, 1] - ev[:-1, 6]).mean()] + [(ev[:, k + 1] - ev[:, k]).mean() for k in range(1, 6)]
    groups.setdefault(rows, []).append([period] + ph)
for rows in sorted(groups):
    v = np.array(groups[rows]).mean(0)
    print(f"  {rows:4d} {len(groups[rows]):5d} " + " ".join(f"{x:8.0f}" for x in v))

# CTA duration by (items, rows of each item, tiles): what the cost model must capture
print("\nCTA duration by shape: n_items rows... tiles -> n, mean dur us")
shape = {}
for c in range(n_cta):
    its = list(range(S["cta_begin"][c], S["cta_begin"][c + 1]))
    key = (len(its), tuple(int(S["items"][i][4]) * ctx.group for i in its), int(t[c, 3]))
    shape.setdefault(key, []).append(dur[c])
for k in sorted(shape, key=lambda k: -np.mean(shape[k])):
    print(f"  {k}: n={len(shape[k])} mean {np.mean(shape[k]):.2f} min {np.min(shape[k]):.2f} max {np.max(shape[k]):.2f}")

# GPU-wide consumption rate over time: each tile's K+V bytes counted when the
# softmax sees its S (clock64 -> ns at the SM clock, anchored at CTA start)
clk_ghz = float(np.median((t[:, 5] - t[:, 4]) / np.maximum(t[:, 1] - t[:, 0], 1)))
print(f"\nSM clock during the launch (clock64 / globaltimer): {clk_ghz:.3f} GHz")
bins = np.zeros(64)
active = np.zeros(64)
for c in range(n_cta):
    nt = min(int(t[c, 3]), NT)
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8)
    b = ev[0, 0]
    tiles = [tt for i in range(S["cta_begin"][c], S["cta_begin"][c + 1])
             for tt in range(int(S["items"][i][1]), int(S["items"][i][2]))]
    for i in range(nt):
        ts = start[c] + (ev[i, 1] - t[c, 4]) / clk_ghz / 1e3
        bins[min(int(ts), 63)] += int(S["tile_ng"][tiles[i]]) * 8192
    for us in range(int(start[c]), min(int(end[c]) + 1, 64)):
        active[us] += 1
n = int(end.max()) + 1
print("\nGPU-wide KV consumption per us (GB/s) and active CTAs:")
print("  " + " ".join(f"{bins[i] / 1e3:5.0f}" for i in range(n)))
print("  " + " ".join(f"{active[i]:5.0f}" for i in range(n)))

# where each CTA's time goes at the start and the end (us, all CTAs)
def us(c, clk):
    return start[c] + (clk - t[c, 4]) / clk_ghz / 1e3
rows_ = []
for c in range(n_cta):
    nt = min(int(t[c, 3]), NT)
    if nt == 0:
        continue
    ev = t[c, 8:8 + 8 * NT].reshape(NT, 8)
    first_s = us(c, ev[0, 1])
    last_p = us(c, ev[nt - 1, 6])
    ofull = us(c, t[c, 248]) if t[c, 248] else np.nan
    stored = us(c, t[c, 250]) if t[c, 250] else np.nan
    xch = us(c, t[c, 252]) if t[c, 252] else np.nan
    wend = max(us(c, x) for x in t[c, 224:232] if x) if any(t[c, 224:232]) else np.nan
    lbeg = us(c, t[c, 251]) if t[c, 251] else np.nan
    ld = [us(c, x) if x else np.nan for x in t[c, 232:236]]
    rows_.append([first_s - start[c], ofull - last_p, xch - ofull, lbeg - xch, ld[0] - lbeg, ld[1] - ld[0], ld[3] - ld[2],
                  stored - ld[3], wend - stored, end[c] - wend, end[c]])
r_ = np.array(rows_)
for nm, col in zip(["start->S(0)", "P(last)->O_full", "O_full->l_xchg", "l_xchg->loop", "loop->ld0", "ld0->ld1", "ld2->ld3", "ld3->stored", "stored->all warps", "warps->end", "end"], r_.T):
    print(f"  {nm:16s} min {np.nanmin(col):6.2f} median {np.nanmedian(col):6.2f} max {np.nanmax(col):6.2f} us")

