"""Device-schedule semantics on the CPU (host-only context).

The schedule is this framework's own layout (units = spans of flatten chunks
x query-slot blocks, per-token rows and slot ranges, direct/partial outputs,
merge lists).  Its correctness contract is the reference's coverage oracle
(partition_test.cpp:27-55): every (query, path token) pair is attended exactly
once, and nothing off the path.  An fp64 interpreter of the schedule must
reproduce naive_attention."""
import numpy as np
import pytest

from oracle import core
from paper_2404_00242_b200 import TreeAttention


def _ctx(G=1, dtype="f32"):
    # bf16 + d_head 128 routes dense chunks to MMA units
    return TreeAttention(device=-1, n_q_heads=G, n_kv_heads=1, d_head=128 if dtype == "bf16" else 16,
                         kv_dtype=dtype)


def _row_map(ctx, snap):
    root, ids, par, cnt = snap
    m = {}
    for node, c in zip(ids, cnt):
        for t in range(int(c)):
            p, s = ctx.token_ref(int(node), t)
            m[p * ctx.page_tokens + s] = (int(node), t)
    return m


def _units(S):
    for u in range(len(S["kind"])):
        tb, nt, sb, ns = (int(x) for x in S["desc"][u])
        yield u, tb, nt, sb, ns


def check_coverage(ctx, tree: core.Tree, bs):
    snap = tree.snapshot()
    S = ctx.schedule(bs)
    rows = _row_map(ctx, snap)
    leaves = list(tree.leaves())
    seen = {}
    slot_units = {}
    for u, tb, nt, sb, ns in _units(S):
        slots = [int(x) for x in S["slot_leaf"][sb:sb + ns]]
        assert slots == sorted(slots) and len(set(slots)) == len(slots)
        used = set()
        for k in range(tb, tb + nt):
            node, tok = rows[int(S["tok_row"][k])]
            b, e = int(S["tok_be"][k]) & 0xFFFF, int(S["tok_be"][k]) >> 16
            assert 0 <= b < e <= ns
            for j in range(b, e):
                li = slots[j]
                used.add(j)
                key = (li, node, tok)
                seen[key] = seen.get(key, 0) + 1
                assert tree.path_tokens(leaves[li]) > 0
        assert used == set(range(ns)), "every slot of a unit attends something"
        for j in range(ns):
            slot_units.setdefault(slots[j], []).append(int(S["slot_part"][sb + j]))
    # exactly once, exactly the path
    for li, leaf in enumerate(leaves):
        path = []
        cur = int(leaf)
        while cur != -1:
            path += [(cur, t) for t in range(tree.token_count(cur))]
            cur = tree.parent(cur)
        got = {(n, t): c for (l, n, t), c in seen.items() if l == li}
        assert set(got) == set(path), li
        assert all(c == 1 for c in got.values()), li
    # outputs: direct writes once, or partials merged
    merged = {int(l): [int(p) for p in S["merge_parts"][S["merge_begin"][i]:S["merge_begin"][i + 1]]]
              for i, l in enumerate(S["merge_leaf"])}
    for li in range(len(leaves)):
        parts = slot_units.get(li, [])
        if len(parts) == 1 and parts[0] < 0:
            assert parts[0] == -1 - li and li not in merged
        else:
            assert all(p >= 0 for p in parts)
            assert sorted(merged[li]) == sorted(parts)
    return S


def interpret(ctx, tree, content, d, h_q, h_kv, bs):
    """fp64 execution of the schedule (unit online softmax + merge)."""
    S = ctx.schedule(bs)
    rows = _row_map(ctx, tree.snapshot())
    leaves = list(tree.leaves())
    G = h_q // h_kv
    L = len(leaves)
    out = np.zeros((L, h_q, d))
    parts = {}
    for u, tb, nt, sb, ns in _units(S):
        slots = [int(x) for x in S["slot_leaf"][sb:sb + ns]]
        for j, li in enumerate(slots):
            q = content.queries[int(leaves[li])].astype(np.float64).reshape(h_q, d)
            toks = []
            for k in range(tb, tb + nt):
                b, e = int(S["tok_be"][k]) & 0xFFFF, int(S["tok_be"][k]) >> 16
                if b <= j < e:
                    toks.append(rows[int(S["tok_row"][k])])
            K = np.stack([content.keys[n][t] for n, t in toks]).astype(np.float64).reshape(-1, h_kv, d)
            V = np.stack([content.values[n][t] for n, t in toks]).astype(np.float64).reshape(-1, h_kv, d)
            hk = np.arange(h_q) // G
            s = np.einsum("thd,hd->ht", K[:, hk], q) / np.sqrt(d)
            m = s.max(1, keepdims=True)
            w = np.exp(s - m)
            o = np.einsum("ht,thd->hd", w / w.sum(1, keepdims=True), V[:, hk])
            lse = (m + np.log(w.sum(1, keepdims=True))).ravel()
            pid = int(S["slot_part"][sb + j])
            if pid < 0:
                out[-1 - pid] = o
            else:
                parts[pid] = (o, lse)
    for i, li in enumerate(S["merge_leaf"]):
        ps = [parts[int(p)] for p in S["merge_parts"][S["merge_begin"][i]:S["merge_begin"][i + 1]]]
        if not ps:
            continue
        M = np.max([p[1] for p in ps], axis=0)
        w = [np.exp(p[1] - M) for p in ps]
        out[int(li)] = sum(wi[:, None] * p[0] for wi, p in zip(w, ps)) / sum(w)[:, None]
    return out.reshape(L, -1)


@pytest.mark.parametrize("rows,span", [(8, 0), (4, 128), (16, 100000), (1, 0), (8, 1)])
def test_coverage_random_trees(rows, span):
    ctx = _ctx(G=1)
    ctx.set_option("fma_max_rows", rows)
    ctx.set_option("span_tokens", span)
    rng = core.Rng(900 + rows + span)
    for trial in range(25):
        t = core.random_tree(rng, max_leaves=70 if trial % 2 else 12, max_node_tokens=40 if trial % 3 else 300,
                             mutation_steps=40)
        ctx.restore(*t.snapshot())
        for bs in (16, 128):
            check_coverage(ctx, t, bs)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_coverage_gqa_groups(dtype):
    for G in (2, 4, 8):
        ctx = _ctx(G=G, dtype=dtype)
        rng = core.Rng(G)
        for trial in range(10):
            t = core.random_tree(rng, max_leaves=40)
            ctx.restore(*t.snapshot())
            S = check_coverage(ctx, t, 128)
            if dtype == "bf16" and len(t.leaves()) * G > 8:
                assert (S["kind"] == 1).any(), "dense chunks go to the MMA path"


def test_coverage_zero_token_and_holders():
    from oracle.make_golden import holder_token_tree
    ctx = _ctx(G=4, dtype="bf16")
    for snap in (holder_token_tree(300, 64), holder_token_tree(1000, 256)):
        t = core.Tree.from_snapshot(snap)
        ctx.restore(*snap)
        check_coverage(ctx, t, 128)


def test_interpreter_matches_oracle():
    rng = core.Rng(77)
    for trial in range(8):
        G = (1, 2, 4)[trial % 3]
        ctx = _ctx(G=G)
        ctx.set_option("fma_max_rows", (4, 8, 16)[trial % 3])
        t = core.random_tree(rng, max_leaves=30, max_tokens=2000, max_node_tokens=150)
        ctx.restore(*t.snapshot())
        c = core.Content.synth(t, 16, trial, qdim=16 * G)
        got = interpret(ctx, t, c, 16, G, 1, 64)
        ref = core.naive_attention(t, c.expanded(16, G, 1), 16, G)
        for i in range(len(ref)):
            if t.path_tokens(int(t.leaves()[i])) > 0:
                assert core.relative_error(got[i], ref[i]) < 1e-12
