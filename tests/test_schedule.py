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

UNUSED = -(1 << 31)


def _ctx(G=1, dtype="f32", n_kv=1):
    # bf16 + d_head 128 selects the tcgen05 kernel's schedule (128-row lanes)
    return TreeAttention(device=-1, n_q_heads=G * n_kv, n_kv_heads=n_kv, d_head=128 if dtype == "bf16" else 16,
                         kv_dtype=dtype)


def _row_map(ctx, snap):
    root, ids, par, cnt = snap
    m = {}
    for node, c in zip(ids, cnt):
        for t in range(int(c)):
            p, s = ctx.token_ref(int(node), t)
            m[p * ctx.page_tokens + s] = (int(node), t)
    return m


def _items(S):
    for i, it in enumerate(S["items"]):
        head, tb, te, sb, ns, ob, lane, flags = (int(x) for x in it)
        yield i, head, tb, te, sb, ns, ob, flags


def _groups(S, t):
    g0 = int(S["tile_grp_begin"][t])
    for g in range(g0, g0 + int(S["tile_ng"][t])):
        info = int(S["grp_info"][g])
        yield g, int(S["grp_row"][g]), info & 0xFF, (info >> 8) & 0xFFF, info >> 20


def check_coverage(ctx, tree: core.Tree, bs):
    snap = tree.snapshot()
    S = ctx.schedule(bs)
    rows = _row_map(ctx, snap)
    leaves = list(tree.leaves())
    n_heads = ctx.n_local_kv_heads
    max_rows = 128 if S["use_mma"] else 16
    cb = S["cta_begin"]
    assert cb[0] == 0 and cb[-1] == len(S["items"]) and np.all(np.diff(cb) >= 0)
    seen = {}
    codes = {}
    tile_use = {}
    for i, head, tb, te, sb, ns, ob, flags in _items(S):
        slots = [int(x) for x in S["slot_leaf"][sb:sb + ns]]
        assert slots == sorted(slots) and len(set(slots)) == len(slots)
        assert 0 < ns and ns * ctx.group <= max_rows and tb < te
        used = set()
        for t in range(tb, te):
            tile_use[(head, t)] = tile_use.get((head, t), 0) + 1
            ng = int(S["tile_ng"][t])
            assert 1 <= ng <= 8
            # TMA boxes: power-of-two runs of full, row-contiguous groups covering 0..ng-1 once
            cover = []
            for bx in S["tile_boxes"][t][:int(S["tile_nbox"][t])]:
                g, sz = int(bx) >> 2, int(bx) & 3
                cover += list(range(g, g + (1 << sz)))
                gs = list(_groups(S, t))
                for k in range(1, 1 << sz):
                    assert gs[g + k - 1][2] == 16 and gs[g + k][1] == gs[g][1] + 16 * k
            assert cover == list(range(ng))
            for g, row0, cnt, b, e in _groups(S, t):
                assert 1 <= cnt <= 16 and 0 <= b < e <= ns
                for k in range(cnt):
                    node, tok = rows[row0 + k]
                    for j in range(b, e):
                        used.add(j)
                        key = (head, slots[j], node, tok)
                        seen[key] = seen.get(key, 0) + 1
        assert bool(flags & 1) == any(int(c) >= 0 for c in S["slot_out"][ob:ob + ns])
        for j in range(ns):
            code = int(S["slot_out"][ob + j])
            if j in used:
                assert code != UNUSED
                codes.setdefault((slots[j], head), []).append((i, code))
            else:
                assert code == UNUSED
    n_tiles = len(S["tile_ng"])
    assert all(tile_use.get((h, t)) == 1 for h in range(n_heads) for t in range(n_tiles))
    # exactly once, exactly the path, for every head
    for li, leaf in enumerate(leaves):
        path = []
        cur = int(leaf)
        while cur != -1:
            path += [(cur, t) for t in range(tree.token_count(cur))]
            cur = tree.parent(cur)
        for h in range(n_heads):
            got = {(n, t): c for (hh, l, n, t), c in seen.items() if l == li and hh == h}
            assert set(got) == set(path), (li, h)
            assert all(c == 1 for c in got.values()), (li, h)
    # outputs: one direct write, or partials merged in one record
    recs = {(int(S["merge_leaf"][m]), int(S["merge_head"][m])): m for m in range(len(S["merge_leaf"]))}
    own, pub = {}, {}
    if S["fused_merge"]:
        for c in range(len(cb) - 1):
            for m in S["cta_own"][S["cta_own_begin"][c]:S["cta_own_begin"][c + 1]]:
                assert int(m) not in own
                own[int(m)] = c
            for m, n in S["cta_pub"][S["cta_pub_begin"][c]:S["cta_pub_begin"][c + 1]]:
                pub[(c, int(m))] = int(n)
        assert set(own) == set(range(len(S["merge_leaf"])))
    for (li, h), ics in codes.items():
        cs = [c for _, c in ics]
        if len(cs) == 1:
            assert cs[0] == -1 - li and (li, h) not in recs
        else:
            m = recs[(li, h)]
            parts = [int(p) for p in S["merge_parts"][S["merge_begin"][m]:S["merge_begin"][m + 1]]]
            assert sorted(parts) == sorted(cs) and all(int(S["part_merge"][p]) == m for p in parts)
            if S["fused_merge"]:
                # every CTA that wrote one of its partials publishes their count
                cta_of = np.searchsorted(cb, [i for i, _ in ics], side="right") - 1
                assert m in own
                for c in set(cta_of):
                    assert pub[(c, m)] == sum(1 for x in cta_of if x == c)
    empty = {(int(l), int(h)) for l, h in S["empty"]}
    assert empty == {(li, h) for li in range(len(leaves)) for h in range(n_heads) if (li, h) not in codes}
    assert all(tree.path_tokens(leaves[li]) == 0 for li, h in empty)
    return S


def interpret(ctx, tree, content, d, h_q, h_kv, bs):
    """fp64 execution of the schedule (item online softmax + merge), one kv head."""
    S = ctx.schedule(bs)
    rows = _row_map(ctx, tree.snapshot())
    leaves = list(tree.leaves())
    G = h_q // h_kv
    L = len(leaves)
    out = np.zeros((L, h_q, d))
    parts = {}
    for i, head, tb, te, sb, ns, ob, flags in _items(S):
        slots = [int(x) for x in S["slot_leaf"][sb:sb + ns]]
        for j, li in enumerate(slots):
            code = int(S["slot_out"][ob + j])
            if code == UNUSED:
                continue
            q = content.queries[int(leaves[li])].astype(np.float64).reshape(h_q, d)
            toks = []
            for t in range(tb, te):
                for g, row0, cnt, b, e in _groups(S, t):
                    if b <= j < e:
                        toks += [rows[row0 + k] for k in range(cnt)]
            K = np.stack([content.keys[n][t] for n, t in toks]).astype(np.float64).reshape(-1, h_kv, d)
            V = np.stack([content.values[n][t] for n, t in toks]).astype(np.float64).reshape(-1, h_kv, d)
            hk = np.arange(h_q) // G
            s = np.einsum("thd,hd->ht", K[:, hk], q) / np.sqrt(d)
            m = s.max(1, keepdims=True)
            w = np.exp(s - m)
            o = np.einsum("ht,thd->hd", w / w.sum(1, keepdims=True), V[:, hk])
            lse = (m + np.log(w.sum(1, keepdims=True))).ravel()
            if code < 0:
                out[-1 - code] = o
            else:
                parts[code] = (o, lse)
    for m_i, li in enumerate(S["merge_leaf"]):
        ps = [parts[int(p)] for p in S["merge_parts"][S["merge_begin"][m_i]:S["merge_begin"][m_i + 1]]]
        M = np.max([p[1] for p in ps], axis=0)
        w = [np.exp(p[1] - M) for p in ps]
        out[int(li)] = sum(wi[:, None] * p[0] for wi, p in zip(w, ps)) / sum(w)[:, None]
    return out.reshape(L, -1)


@pytest.mark.parametrize("rows,ctas", [(8, 148), (4, 7), (16, 1), (1, 148), (8, 1000)])
def test_coverage_random_trees(rows, ctas):
    ctx = _ctx(G=1)
    ctx.set_option("use_mma", 0)
    ctx.set_option("fma_max_rows", rows)
    ctx.set_option("num_ctas", ctas)
    rng = core.Rng(900 + rows + ctas)
    for trial in range(25):
        t = core.random_tree(rng, max_leaves=70 if trial % 2 else 12, max_node_tokens=40 if trial % 3 else 300,
                             mutation_steps=40)
        ctx.restore(*t.snapshot())
        for bs in (16, 128):
            check_coverage(ctx, t, bs)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_coverage_gqa_groups(dtype):
    for G in (2, 4, 8):
        ctx = _ctx(G=G, dtype=dtype, n_kv=3)
        ctx.set_option("num_ctas", 37)
        rng = core.Rng(G)
        for trial in range(10):
            t = core.random_tree(rng, max_leaves=40)
            ctx.restore(*t.snapshot())
            S = check_coverage(ctx, t, 128)
            assert S["use_mma"] == (dtype == "bf16")


def test_coverage_wide_stripes_mma():
    """>128 rows: wide stripes split into balanced slot blocks (MMA lanes)."""
    ctx = _ctx(G=4, dtype="bf16", n_kv=2)
    rng = core.Rng(5)
    for trial in range(6):
        t = core.random_tree(rng, max_leaves=120, max_node_tokens=200)
        ctx.restore(*t.snapshot())
        S = check_coverage(ctx, t, 128)
    t = core.Tree(4000)
    kids = t.branch(t.root, [0] * 50)
    for k in kids:
        t.append_tokens(k, 400)
    ctx.restore(*t.snapshot())
    S = check_coverage(ctx, t, 128)
    assert S["n_lanes"] >= 2


def test_coverage_zero_token_and_holders():
    from oracle.make_golden import holder_token_tree
    ctx = _ctx(G=4, dtype="bf16")
    for snap in (holder_token_tree(300, 64), holder_token_tree(1000, 256)):
        t = core.Tree.from_snapshot(snap)
        ctx.restore(*snap)
        check_coverage(ctx, t, 128)


def test_coverage_item_cost_repartition():
    """The re-partition with the higher item cost (CTAs with many items), the
    per-box tile cost and both CTA partitions keep the coverage contract."""
    rng = core.Rng(404)
    for trial in range(6):
        ctx = _ctx(G=4, dtype="bf16", n_kv=2)
        ctx.set_option("many_items", 1)          # always re-partition
        ctx.set_option("item_cost_many", (450, 5000)[trial % 2])
        ctx.set_option("num_ctas", (13, 148)[trial % 2])
        ctx.set_option("minmax", trial % 3 != 2)   # min-max budget / equal split points
        ctx.set_option("box_cost", (0, 40, 0)[trial % 3])   # per-box term of the tile cost
        t = core.random_tree(rng, max_leaves=50, max_node_tokens=200)
        ctx.restore(*t.snapshot())
        check_coverage(ctx, t, 128)


def test_interpreter_fused_merge_matches_oracle():
    """tcgen05 schedules (bf16, d 128) merge split leaf-heads in their last
    item: the interpreter with owner shares reproduces naive_attention."""
    rng = core.Rng(78)
    for trial in range(4):
        ctx = _ctx(G=4, dtype="bf16")
        ctx.set_option("num_ctas", (5, 37, 148, 148)[trial])
        t = core.random_tree(rng, max_leaves=40, max_tokens=3000, max_node_tokens=300)
        ctx.restore(*t.snapshot())
        S = ctx.schedule(128)
        assert S["fused_merge"]
        c = core.Content.synth(t, 128, trial, qdim=128 * 4)
        got = interpret(ctx, t, c, 128, 4, 1, 128)
        ref = core.naive_attention(t, c.expanded(128, 4, 1), 128, 4)
        for i in range(len(ref)):
            if t.path_tokens(int(t.leaves()[i])) > 0:
                assert core.relative_error(got[i], ref[i]) < 1e-12


def test_interpreter_matches_oracle():
    rng = core.Rng(77)
    for trial in range(8):
        G = (1, 2, 4)[trial % 3]
        ctx = _ctx(G=G)
        ctx.set_option("fma_max_rows", (4, 8, 16)[trial % 3])
        ctx.set_option("num_ctas", (3, 50, 148)[trial % 3])
        t = core.random_tree(rng, max_leaves=30, max_tokens=2000, max_node_tokens=150)
        ctx.restore(*t.snapshot())
        c = core.Content.synth(t, 16, trial, qdim=16 * G)
        got = interpret(ctx, t, c, 16, G, 1, 64)
        ref = core.naive_attention(t, c.expanded(16, G, 1), 16, G)
        for i in range(len(ref)):
            if t.path_tokens(int(t.leaves()[i])) > 0:
                assert core.relative_error(got[i], ref[i]) < 1e-12
