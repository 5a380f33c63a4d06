"""GPU parity at every benchmarked configuration (BASELINE.json configs), at
full size, through the C ABI.

Each test builds the bench's own tree (bench.build_snapshot: the reference's
generators gen_few_shot / reasoning records / gen_speculative, workloads.hpp),
fills it with the reference's synthetic content (synth.hpp:41-69, rounded to
bf16 as SURVEY §8c item 2 prescribes) and compares every leaf and every head
with the fp64 dense reference (naive_attention, attention.hpp:237-288, with the
tree mask as the ancestor relation, partition.hpp:267-279).

Gates (north_star): bf16 with fp32 accumulation within 2e-2 max-abs AND the
reference's relative_error (attention.hpp:337-346) <= 1e-2 per leaf (the
relative gate keeps the absolute bound non-vacuous on flat softmaxes); fp32
within 1e-5 relative_error."""
import numpy as np
import pytest

import bench
from gpu_helpers import dense_reference, load_into, make_content, q_tensor
from oracle import core

pytestmark = pytest.mark.gpu

BF16_ABS, BF16_REL = 2e-2, 1e-2


def _ctx(snap, d, h_q, h_kv, kv_dtype="bf16", kv_head_begin=0, n_local=0, options=None, n_layers=1):
    from paper_2404_00242_b200 import TreeAttention
    root, ids, par, cnt = snap
    pages = int(sum((int(c) + 15) // 16 for c in cnt)) + 8
    ctx = TreeAttention(n_layers=n_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype=kv_dtype,
                        out_dtype="f32", max_pages=pages, device=0, kv_head_begin=kv_head_begin,
                        n_local_kv_heads=n_local)
    for k, v in (options or {}).items():
        ctx.set_option(k, v)
    ctx.restore(*snap)
    return ctx


def _attend(ctx, content, q_head_begin=0, content_kv_head=0, layer=0):
    import torch
    load_into(ctx, content, layer=layer, kv_head_begin=content_kv_head)
    leaves = ctx.leaves()
    q = q_tensor(ctx, content, leaves, q_head_begin=q_head_begin)
    lse = torch.full((len(leaves), ctx.n_local_q_heads), float("nan"), device="cuda")
    ctx.prepare(128)
    out = ctx.attend(layer, q, lse=lse)
    torch.cuda.synchronize()
    return out.float().cpu().numpy().astype(np.float64).reshape(len(leaves), -1), lse.cpu().numpy(), leaves


def _check(out, lse, ref, ref_lse, what):
    err = np.abs(out - ref)
    assert np.isfinite(out).all(), what
    assert err.max() <= BF16_ABS, (what, float(err.max()))
    worst = max(core.relative_error(out[i], ref[i]) for i in range(ref.shape[0]))
    assert worst <= BF16_REL, (what, worst)
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(lse), fin), what
    np.testing.assert_allclose(lse[fin], ref_lse[fin], atol=2e-2, err_msg=what)
    return worst


def _full_config(name, seed=42, options=None):
    cfg = bench.CONFIGS[name]
    snap = bench.build_snapshot(cfg)
    t = core.Tree.from_snapshot(snap)
    c = make_content(t, cfg["d"], cfg["h_q"], cfg["h_kv"], seed, bf16=True)
    ctx = _ctx(snap, cfg["d"], cfg["h_q"], cfg["h_kv"], options=options)
    out, lse, leaves = _attend(ctx, c)
    ref, ref_lse = dense_reference(snap, c, cfg["d"], cfg["h_q"], cfg["h_kv"], leaves)
    return ctx, _check(out, lse, ref, ref_lse, name)


def test_config_b_few_shot_all_leaves():
    """Config B (gen_few_shot(4000, 50, 400) iteration 400): every leaf, every head."""
    ctx, _ = _full_config("few_shot")
    io = ctx.io_stats()
    assert io.kv_bytes == 24000 * 2 * 8 * 128 * 2


def test_config_c_reasoning_standin():
    """Config C: the ToT stand-in (N = 37,365, 65 nodes, 55 leaves, depth 11)."""
    ctx, _ = _full_config("reasoning")
    assert ctx.info()["total_tokens"] == 37365
    assert len(ctx.leaves()) == 55


def test_config_d_spec_t64_p4k():
    """Config D: token tree t = 64 over a 4k prompt (64 queries via holders)."""
    _full_config("spec_t64")


def test_config_d_spec_t256_p16k():
    """Config D: token tree t = 256 over a 16k prompt: ~1,000 rows per kv head,
    8 lanes per wide stripe, thousands of partials."""
    ctx, _ = _full_config("spec_t256")
    assert ctx.io_stats().n_partials > 1000


@pytest.mark.parametrize("kv_head", [0, 5])
def test_config_e_70b_per_gpu_shard(kv_head):
    """Config E's per-GPU shard at 8 GPUs: h_q 64 / h_kv 8 (G = 8), one kv head
    and its 8 q heads, gen_few_shot(32000, 50, 400) iteration 400 (N = 52,000)."""
    cfg = bench.CONFIGS["few_shot_70b"]
    snap = bench.build_snapshot(cfg)
    t = core.Tree.from_snapshot(snap)
    assert t.total_tokens() == 52000
    # content of this shard only: one kv head (d) and its G = 8 query heads
    c = core.Content.synth(t, 128, 700 + kv_head, qdim=8 * 128).map(core.bf16_round)
    ctx = _ctx(snap, 128, 64, 8, kv_head_begin=kv_head, n_local=1)
    assert ctx.n_local_q_heads == 8
    out, lse, leaves = _attend(ctx, c)
    ref, ref_lse = dense_reference(snap, c, 128, 8, 1, leaves)
    _check(out, lse, ref, ref_lse, f"70B shard {kv_head}")


def test_head_sharding_on_one_gpu():
    """Head sharding with two contexts on cuda:0 owning kv heads
    [0, 4) and [4, 8): their outputs side by side equal the unsharded oracle,
    with no collective."""
    snap = bench.build_snapshot(dict(kind="few_shot", prefix=1500, branches=20, iteration=90))
    t = core.Tree.from_snapshot(snap)
    c = make_content(t, 128, 32, 8, 77, bf16=True)
    parts, lses = [], []
    for begin in (0, 4):
        ctx = _ctx(snap, 128, 32, 8, kv_head_begin=begin, n_local=4)
        out, lse, leaves = _attend(ctx, c, q_head_begin=begin * 4, content_kv_head=begin)
        parts.append(out)
        lses.append(lse)
    full, full_lse = np.concatenate(parts, axis=1), np.concatenate(lses, axis=1)
    ref, ref_lse = dense_reference(snap, c, 128, 32, 8, leaves)
    _check(full, full_lse, ref, ref_lse, "head shards")
    ctx = _ctx(snap, 128, 32, 8)
    out, _, _ = _attend(ctx, c)
    assert np.max(np.abs(out - full)) <= 1e-2


def test_fma_group_of_16():
    """FMA kernel with G = 16 > fma_max_rows (fp32, h_q 32 / h_kv 2): lanes of
    one slot carry 16 rows; every q head must be computed."""
    t = core.Tree(700)
    kids = t.branch(t.root, [90, 0, 33, 250])
    t.branch(kids[2], [5, 61])
    snap = t.snapshot()
    c = make_content(t, 64, 32, 2, 3, bf16=False)
    for rows in (4, 8, 16):
        ctx = _ctx(snap, 64, 32, 2, kv_dtype="f32", options={"fma_max_rows": rows})
        out, lse, leaves = _attend(ctx, c)
        ref, _ = dense_reference(snap, c, 64, 32, 2, leaves)
        for i in range(len(leaves)):
            assert core.relative_error(out[i], ref[i]) <= 1e-5, (rows, i)


def test_fma_group_too_large_rejected():
    """G = 32 exceeds the FMA kernel's rows: a clear invalid_argument."""
    t = core.Tree(50)
    t.branch(t.root, [3, 4])
    ctx = _ctx(t.snapshot(), 64, 32, 1, kv_dtype="f32")
    with pytest.raises(ValueError, match="group size"):
        ctx.prepare(128)


def test_bf16_fma_and_mma_agree_on_70b_shape():
    """The FMA kernel (use_mma = 0) on the G = 8 shape agrees with the oracle
    too (per-item kernel choice needs both paths right on the same schedule)."""
    snap = bench.build_snapshot(dict(kind="few_shot", prefix=2000, branches=10, iteration=50))
    t = core.Tree.from_snapshot(snap)
    c = core.Content.synth(t, 128, 5, qdim=8 * 128).map(core.bf16_round)
    for opts in ({"use_mma": 0}, {}):
        ctx = _ctx(snap, 128, 64, 8, kv_head_begin=2, n_local=1, options=opts)
        out, lse, leaves = _attend(ctx, c)
        ref, ref_lse = dense_reference(snap, c, 128, 8, 1, leaves)
        _check(out, lse, ref, ref_lse, str(opts))
