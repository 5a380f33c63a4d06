"""The reference's other partition strategies and its IO model, on the host
(no GPU).

* make_plan for Node / Node-Chunk / Q-guided (partition.hpp:133-207) is
  byte-identical to the reference's plan_to_json (compiled reference when
  available, oracle/_ref).
* io_measured / io_analytical (io_model.hpp:88-170) equal the reference's
  numbers: the committed golden fixtures (tests/golden/io.json) and, when the
  compiled reference is present, random trees for every algorithm."""
import numpy as np
import pytest

import golden_io as G
from oracle import core, ref
from paper_2404_00242_b200 import TreeAttention

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref (compiled reference) not built")


def _ctx(snap):
    ctx = TreeAttention(device=-1, n_q_heads=4, n_kv_heads=1, d_head=16)
    ctx.restore(*snap)
    return ctx


def test_io_golden_fixtures():
    """io.json: io_measured(partition_flatten) and io_analytical(Flatten,
    FlashDecoding) of the compiled reference, CostParams{128, 32, 32, 2}."""
    for case in G.io():
        ctx = _ctx(G.snap(case["tree"]))
        assert list(ctx.io_measured(128, 128, 32, 32, 2)) == case["measured"], case["name"]
        assert list(ctx.io_analytical("flatten", 128, 128, 32, 32, 2)) == case["flatten"], case["name"]
        assert list(ctx.io_analytical("flash-decoding", 128, 128, 32, 32, 2)) == case["flash_decoding"], case["name"]


@needs_ref
@pytest.mark.parametrize("strategy", ["node", "node-chunk", "q-guided", "flatten"])
def test_strategy_plans_bit_exact(strategy):
    snaps = ref.random_trees(4321, 30, max_leaves=90, max_node_tokens=300, mutation_steps=40)
    snaps += [ref.few_shot(600, 5, 30)[29], ref.preset("fig2")[0]]
    from oracle.make_golden import holder_token_tree
    snaps += [holder_token_tree(200, 64)]
    for s in snaps:
        ctx = _ctx(s)
        ctx.set_strategy(strategy)
        for bs in (7, 32, 128):
            assert ctx.plan_json(bs) == ref.plan_json(s, bs, strategy), (strategy, bs)


@needs_ref
def test_io_model_matches_reference_random_trees():
    algs = ["naive", "flash-decoding", "radix", "tree-attn-medusa", "tree-attn-specinfer", "node", "node-chunk",
            "flatten"]
    for s in ref.random_trees(77, 25, max_leaves=100, max_node_tokens=200, mutation_steps=40):
        ctx = _ctx(s)
        for bs in (16, 128):
            for params in ((128, 32, 32, 2), (64, 8, 80, 4)):
                for a in algs:
                    assert ctx.io_analytical(a, bs, *params) == ref.io_analytical(s, a, bs, *params), a
                for st in ("flatten", "node", "node-chunk", "q-guided"):
                    ctx.set_strategy(st)
                    assert ctx.io_measured(bs, *params) == ref.io_measured(s, bs, *params, strategy=st), st
                ctx.set_strategy("flatten")


def test_strategy_schedules_cover_the_tree():
    """Each ablation plan on the device schedule: every (leaf, path token) is
    attended exactly once per head (the same coverage contract as flatten)."""
    import test_schedule as TS
    rng = core.Rng(31337)
    for trial in range(6):
        t = core.random_tree(rng, max_leaves=40, max_node_tokens=200)
        for strategy in ("node", "node-chunk", "q-guided"):
            for dtype, G_ in (("bf16", 4), ("f32", 1)):
                ctx = TS._ctx(G=G_, dtype=dtype, n_kv=2)
                ctx.set_strategy(strategy)
                ctx.restore(*t.snapshot())
                TS.check_coverage(ctx, t, 64)


def test_q_guided_loads_every_path():
    """Q-guided loads each leaf's whole path (sum of path lengths, the F_s-fold
    KV IO that DeFT removes); flatten loads the tree once."""
    t = core.Tree(1000)
    kids = t.branch(t.root, [50] * 6)
    ctx = TreeAttention(device=-1, n_q_heads=4, n_kv_heads=1, d_head=128, kv_dtype="bf16")
    ctx.restore(*t.snapshot())
    S = ctx.schedule(128)
    flat_rows = sum(int(S["tile_ng"][i]) for i in range(len(S["tile_ng"])))
    ctx.set_strategy("q-guided")
    S = ctx.schedule(128)
    qg_rows = sum(int(S["tile_ng"][i]) for i in range(len(S["tile_ng"])))
    assert qg_rows >= 4 * flat_rows   # F_s = 6300 / 1300
