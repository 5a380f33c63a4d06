"""TMA box-size histogram of each bench config's schedule (16/32/64/128-row boxes)."""
import sys; sys.path.insert(0,'.')
import numpy as np, bench
from paper_2404_00242_b200 import TreeAttention
for name in ["few_shot","reasoning","spec_t64","spec_t256","few_shot_70b_shard"]:
    cfg=dict(bench.CONFIGS[name]); snap=bench.build_snapshot(cfg); root,ids,par,cnt=snap
    n_loc=cfg.get("n_local_kv_heads") or cfg["h_kv"]
    ctx=TreeAttention(n_layers=1,n_q_heads=cfg["h_q"],n_kv_heads=cfg["h_kv"],d_head=cfg["d"],kv_dtype="bf16",out_dtype="bf16",
        max_pages=int(sum((int(c)+15)//16 for c in cnt))+16,n_local_kv_heads=n_loc)
    ctx.restore(*snap)
    try:
        ctx.prepare(128)
    except Exception as e:
        print(name, "prepare failed", e); continue
    S=ctx.schedule(128)
    nb=S["tile_nbox"]; bx=S["tile_boxes"]
    hist=np.zeros(4,int)
    for t in range(len(nb)):
        for b in bx[t][:nb[t]]: hist[int(b)&3]+=1
    heads=n_loc
    print(f"{name}: tiles/head {len(nb)}, boxes by size (16,32,64,128 rows) per head {hist.tolist()}, TMA instr per layer (K+V, 2 halves) {4*hist.sum()*heads}, bytes {sum(hist*np.array([16,32,64,128]))*512*heads/1e6:.1f} MB")
