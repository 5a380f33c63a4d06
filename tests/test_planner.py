"""Host side of the product (no GPU): the tree mirror, page accounting and the
bit-exact flatten planner of libtreeattn_b200.so, against the reference's
golden plans and against the oracle restatement.  Reference tests mirrored:
tree_test.cpp, kv_cache_test.cpp, partition_test.cpp."""
import numpy as np
import pytest

import golden_io as G
from oracle import core
from paper_2404_00242_b200 import InvalidArgument, LogicError, OutOfRange, TreeAttention


@pytest.fixture
def ctx():
    c = TreeAttention(device=-1, n_q_heads=1, d_head=16)
    yield c
    c.close()


def test_golden_plans_bit_exact(ctx):
    for case in G.plans():
        ctx.restore(*G.snap(case["tree"]))
        assert ctx.plan_json(case["block_size"]) == case["plan"], (case["name"], case["block_size"])


def test_plans_match_oracle_on_random_trees(ctx):
    rng = core.Rng(4242)
    for trial in range(120):
        kw = dict(max_leaves=80 if trial % 2 else 20, max_node_tokens=30 if trial % 3 == 0 else 200,
                  mutation_steps=60)
        t = core.random_tree(rng, **kw)
        ctx.restore(*t.snapshot())
        for bs in (1, 7, 64, 128):
            assert ctx.plan_json(bs) == core.plan_to_json(core.partition_flatten(t, bs)), (trial, bs)


def test_plan_view_matches_json(ctx):
    ctx.new_tree(4)
    ctx.branch(0, [2, 2])
    p = ctx.plan_flatten(6)
    assert core.plan_to_json(p) == ctx.plan_json(6)
    assert p["groups"][0]["masks"] == [0b11, 0b01]


def test_plan_block_size_error(ctx):
    ctx.new_tree(10)
    with pytest.raises(InvalidArgument):
        ctx.plan_json(0)


# ---- DecodingTree semantics (tree_test.cpp) --------------------------------
def test_tree_basics(ctx):
    r = ctx.new_tree(4000)
    assert list(ctx.leaves()) == [r]
    kids = ctx.branch(r, [400, 400])
    assert ctx.info()["total_tokens"] == 4800
    assert set(ctx.leaves()) == set(kids)
    with pytest.raises(OutOfRange):
        ctx.branch(9999, [1])
    with pytest.raises(InvalidArgument):
        ctx.branch(r, [1])
    with pytest.raises(InvalidArgument):
        ctx.new_tree(0)


def test_deep_wide_branching(ctx):
    frontier = ctx.new_tree(1000)
    for _ in range(10):
        frontier = ctx.branch(frontier, [100] * 10)[0]
    assert ctx.info()["node_count"] == 101
    assert len(ctx.leaves()) == 91


def test_prune_and_append(ctx):
    r = ctx.new_tree(10)
    kids = ctx.branch(r, [5, 7])
    ctx.prune(kids[1])
    assert len(ctx.leaves()) == 1 and ctx.info()["total_tokens"] == 15
    with pytest.raises(InvalidArgument):
        ctx.prune(r)
    with pytest.raises(OutOfRange):
        ctx.prune(kids[1])
    ctx.append_tokens(kids[0], 3)
    assert ctx.info()["total_tokens"] == 18
    with pytest.raises(InvalidArgument):
        ctx.append_tokens(r, 1)
    with pytest.raises(InvalidArgument):
        ctx.append_tokens(kids[0], 0)
    # ids are never reused
    assert ctx.branch(kids[0], [1])[0] == 3


def test_leaves_dfs_order_matches_oracle(ctx):
    rng = core.Rng(42)
    for _ in range(30):
        t = core.random_tree(rng)
        ctx.restore(*t.snapshot())
        assert list(ctx.leaves()) == list(t.leaves())
        assert ctx.info()["path_tokens_sum"] == sum(t.path_tokens(l) for l in t.leaves())


def test_restore_errors(ctx):
    with pytest.raises(InvalidArgument):  # duplicate id
        ctx.restore(0, [0, 1, 1], [-1, 0, 0], [1, 1, 1])
    with pytest.raises(InvalidArgument):  # dangling parent
        ctx.restore(0, [0, 1], [-1, 7], [1, 1])
    with pytest.raises(InvalidArgument):  # root with parent
        ctx.restore(0, [0, 1], [1, 0], [1, 1])


# ---- PagePool accounting (kv_cache_test.cpp) -------------------------------
def test_page_ceiling_division(ctx):
    ctx.new_tree(4000)
    assert ctx.pool_stats()["page_count"] == 250
    ctx.new_tree(17)
    assert ctx.pool_stats()["page_count"] == 2


def test_pages_never_shared_and_recycled(ctx):
    r = ctx.new_tree(3)
    a, b = ctx.branch(r, [3, 3])
    st = ctx.pool_stats()
    assert st["page_count"] == 3 and st["live_slots"] == 9
    ctx.prune(b)
    st = ctx.pool_stats()
    assert st["free_page_count"] == 1 and st["live_slots"] == 6
    c = ctx.branch(a, [10])[0]
    st = ctx.pool_stats()
    assert st["page_count"] == 3 and st["free_page_count"] == 0  # recycled
    assert ctx.token_ref(c, 0)[0] != ctx.token_ref(a, 0)[0]


def test_extend_fills_tail_first(ctx):
    r = ctx.new_tree(10)
    ctx.append_tokens(r, 6)
    assert ctx.pool_stats()["page_count"] == 1
    ctx.append_tokens(r, 1)
    assert ctx.pool_stats()["page_count"] == 2
    assert ctx.token_ref(r, 15) == (0, 15) and ctx.token_ref(r, 16) == (1, 0)
    with pytest.raises(InvalidArgument):
        ctx.token_ref(r, 17)


def test_accounting_invariant_random(ctx):
    rng = core.Rng(11)
    t = core.random_tree(rng)
    ctx.restore(*t.snapshot())
    assert ctx.pool_stats()["live_slots"] == t.total_tokens()
    leaf = int(ctx.leaves()[-1])
    if leaf != ctx.info()["root"]:
        before = ctx.pool_stats()["live_slots"]
        drop = t.token_count(leaf)
        ctx.prune(leaf)
        assert ctx.pool_stats()["live_slots"] == before - drop


def test_host_only_context_refuses_attention(ctx):
    from paper_2404_00242_b200 import NoDevice
    ctx.new_tree(10)
    with pytest.raises(NoDevice):
        ctx.prepare(128)
