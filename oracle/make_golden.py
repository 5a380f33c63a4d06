"""Generate tests/golden/ fixtures from the REAL reference (oracle/_ref).

Run in the build container (needs /root/reference to build _ref):
    python -m oracle.make_golden

Fixtures are small and committed; the GPU box never needs /root/reference.
Contents:
  rng.json        fill_uniform vectors, content_seed values, random_tree
                  snapshots (synth.hpp:20-111) -- pins the C restatement
  plans.json.gz   plan_to_json(partition_flatten(tree, bs)) for the
                  reference's own golden trees (partition_test.cpp), random
                  trees, presets and 0-token-holder token trees
  attention.npz   run_iteration (float and double engines) and naive_attention
                  outputs for small synth instances (attention_test.cpp style)
  io.json         io_measured / io_analytical(Flatten, FlashDecoding)
"""
from __future__ import annotations

import gzip
import json
import os

import numpy as np

from . import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")


def snap_obj(s):
    root, ids, par, cnt = s
    return {"root": int(root), "ids": [int(x) for x in ids], "parents": [int(x) for x in par],
            "counts": [int(x) for x in cnt]}


def chain_snap(counts, parents):
    ids = list(range(len(counts)))
    return (0, np.array(ids, np.int32), np.array(parents, np.int32), np.array(counts, np.int64))


def holder_token_tree(prompt, t):
    """gen_speculative's token tree (workloads.hpp:192-205, 218-271) with one
    0-token query holder under every interior token node."""
    topo = []
    remaining, head = t, -1
    while remaining > 0:
        width = max(1, remaining // 2)
        first = len(topo)
        topo += [head] * width
        head = first
        remaining -= width
    ids, par, cnt = [0], [-1], [prompt]
    tree_id = {}
    nxt = 1
    children = {}
    for i, p in enumerate(topo):
        children.setdefault(p, []).append(i)
    def add(node_parent, cnt_):
        nonlocal nxt
        ids.append(nxt); par.append(node_parent); cnt.append(cnt_)
        nxt += 1
        return nxt - 1
    # graft level by level like gen_speculative; interior nodes get a holder
    for i in children.get(-1, []):
        tree_id[i] = add(0, 1)
    for i in range(t):
        kids = children.get(i, [])
        if kids:
            for k in kids:
                tree_id[k] = add(tree_id[i], 1)
            add(tree_id[i], 0)  # 0-token query holder
    return (0, np.array(ids, np.int32), np.array(par, np.int32), np.array(cnt, np.int64))


def main():
    assert ref.available(), "build oracle/_ref first (make -C oracle ref)"
    os.makedirs(OUT, exist_ok=True)

    # ---------------------------------------------------------------- rng
    rng = {"fill_uniform": [], "content_seed": [], "random_trees": {}}
    for seed in [0, 1, 42, 12345, 2**63 + 7]:
        rng["fill_uniform"].append({"seed": seed, "v": [float(x) for x in ref.fill_uniform(64, seed)]})
    for (s, a, b) in [(42, 0, 0), (42, 7, 13), (2024, 1, 2**40), (0xabcdef12, 3, 0)]:
        rng["content_seed"].append({"args": [s, a, b], "value": str(ref.content_seed(s, a, b))})
    for key, kw in {"seed2024_d60_s12": dict(seed=2024, n=40, max_node_tokens=60, mutation_steps=12),
                    "seed23_default": dict(seed=23, n=20),
                    "seed71_max2048": dict(seed=71, n=20, max_tokens=2048)}.items():
        seed, n = kw.pop("seed"), kw.pop("n")
        rng["random_trees"][key] = {"seed": seed, "n": n, "cfg": kw,
                                    "snaps": [snap_obj(s) for s in ref.random_trees(seed, n, **kw)]}
    with open(os.path.join(OUT, "rng.json"), "w") as f:
        json.dump(rng, f)

    # -------------------------------------------------------------- plans
    cases = []

    def add(name, snap, bss):
        for bs in bss:
            cases.append({"name": name, "block_size": bs, "tree": snap_obj(snap), "plan": ref.plan_json(snap, bs)})

    # partition_test.cpp golden trees
    add("hand_5_3_4", chain_snap([5, 3, 4], [-1, 0, 1]), [4, 1, 3, 128])
    add("exact_4096", chain_snap([4096], [-1]), [128])
    add("fig2", ref.preset("fig2")[0], [6, 1, 2, 4, 128])
    add("star70", (0, np.arange(71, dtype=np.int32), np.array([-1] + [0] * 70, np.int32),
                   np.array([100] + [5] * 70, np.int64)), [64, 128])
    add("zero_token", (0, np.arange(3, dtype=np.int32), np.array([-1, 0, 0], np.int32),
                       np.array([10, 0, 5], np.int64)), [4])
    add("demo", (0, np.arange(5, dtype=np.int32), np.array([-1, 0, 0, 0, 0], np.int32),
                 np.array([1024, 128, 128, 128, 128], np.int64)), [128])
    for i, s in enumerate(ref.random_trees(23, 12)):
        add(f"random23_{i}", s, [16, 64, 128])
    for i, s in enumerate(ref.random_trees(99, 6, max_leaves=200, max_node_tokens=50, mutation_steps=160)):
        add(f"random_wide_{i}", s, [16, 128])
    fs = ref.few_shot(4000, 50, 400)
    for it in [1, 200, 400]:
        add(f"few_shot_b50_it{it}", fs[it - 1], [128])
    sorting = ref.preset("sorting")
    peak = max(range(len(sorting)), key=lambda i: int(sorting[i][3].sum()))
    add("sorting_peak", sorting[peak], [128])
    for t in [32, 64, 128, 256]:
        add(f"spec_t{t}_p4k", ref.spec({"kind": "speculative", "prompt_len": 4000, "tree_size": t, "steps": 1})[0], [128])
    add("spec_t256_p16k", ref.spec({"kind": "speculative", "prompt_len": 16000, "tree_size": 256, "steps": 1})[0], [128])
    for t in [32, 64]:
        add(f"holder_t{t}", holder_token_tree(4000, t), [128, 16])
    with gzip.open(os.path.join(OUT, "plans.json.gz"), "wt") as f:
        json.dump(cases, f)

    # ---------------------------------------------------------- attention
    arrays = {}
    meta = []
    att_cases = []
    for i, s in enumerate(ref.random_trees(2024, 6, max_node_tokens=60, mutation_steps=12)):
        att_cases.append((f"rt2024_{i}", s, 16, 2, 1000 + i, 32))
    for i, s in enumerate(ref.random_trees(7, 3, max_tokens=1500)):
        att_cases.append((f"rt7_d64_{i}", s, 64, 1, 500 + i, 128))
    att_cases.append(("fig2_d8", ref.preset("fig2")[0], 8, 1, 5, 6))
    att_cases.append(("hand_5_3_4", chain_snap([5, 3, 4], [-1, 0, 1]), 16, 2, 3, 4))
    att_cases.append(("zero_token", (0, np.arange(3, dtype=np.int32), np.array([-1, 0, 0], np.int32),
                                     np.array([10, 0, 5], np.int64)), 16, 1, 9, 4))
    for name, s, d, h, seed, bs in att_cases:
        inst = ref.Instance.synth(s, d, h, seed)
        of, pf, _ = inst.run_iteration(bs, use_double=False)
        od, pd, _ = inst.run_iteration(bs, use_double=True)
        on, _ = inst.naive()
        arrays[name + "/float"] = of
        arrays[name + "/double"] = od
        arrays[name + "/naive"] = on
        arrays[name + "/present"] = pf.astype(np.uint8)
        meta.append({"name": name, "tree": snap_obj(s), "d_head": d, "n_heads": h, "seed": seed, "block_size": bs})
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **arrays)
    with open(os.path.join(OUT, "attention.json"), "w") as f:
        json.dump(meta, f)

    # ------------------------------------------------------------------ io
    io = []
    for name, s in [("fig2", ref.preset("fig2")[0]), ("few_shot_b50_it400", fs[399]),
                    ("spec_t128", ref.spec({"kind": "speculative", "prompt_len": 4000, "tree_size": 128, "steps": 1})[0])]:
        io.append({"name": name, "tree": snap_obj(s),
                   "measured": list(ref.io_measured(s, 128, 128, 32, 32, 2)),
                   "flatten": list(ref.io_analytical(s, "flatten", 128, 128, 32, 32, 2)),
                   "flash_decoding": list(ref.io_analytical(s, "flash-decoding", 128, 128, 32, 32, 2))})
    with open(os.path.join(OUT, "io.json"), "w") as f:
        json.dump(io, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
