"""§8(f1): the decode step -- batched appends, the step's KV written on the
device, re-planning every step, and a CUDA graph of the layer calls that stays
valid across re-plans.

Reference: gen_few_shot's loop (workloads.hpp:98-111) calls append_tokens
(tree.hpp:119-129) on every leaf, and each new token's KV is written with
PagePool::write_kv (kv_cache.hpp:104-116) before run_iteration."""
import numpy as np
import pytest

from oracle import core
from paper_2404_00242_b200 import TreeAttention


def _few_shot(prefix, branches, it):
    t = core.Tree(prefix)
    kids = t.branch(t.root, [0] * branches)
    for _ in range(it):
        for k in kids:
            t.append_tokens(k, 1)
    return t


# ------------------------------------------------------------------ CPU
def test_append_leaves_matches_sequential_appends():
    """One append_leaves call == append_tokens on every leaf: same tree, same
    bit-exact plan as the reference restatement after the same steps."""
    ref = _few_shot(300, 7, 0)
    ctx = TreeAttention(device=-1, n_q_heads=4, n_kv_heads=1, d_head=16)
    ctx.restore(*ref.snapshot())
    for step in range(40):
        ctx.append_leaves()
        for leaf in ref.leaves():
            ref.append_tokens(int(leaf), 1)
        if step % 13 == 0:
            assert ctx.plan_json(32) == core.plan_to_json(core.partition_flatten(ref, 32))
    assert ctx.plan_json(128) == core.plan_to_json(core.partition_flatten(ref, 128))
    # explicit leaves and counts
    leaves = ctx.leaves()
    ctx.append_leaves(leaves[::2], [3] * len(leaves[::2]))
    for leaf in leaves[::2]:
        ref.append_tokens(int(leaf), 3)
    assert ctx.plan_json(64) == core.plan_to_json(core.partition_flatten(ref, 64))


def test_append_leaves_all_or_nothing():
    ctx = TreeAttention(device=-1, n_q_heads=2, n_kv_heads=2, d_head=16)
    root = ctx.new_tree(10)
    kids = ctx.branch(root, [2, 3])
    snap = ctx.snapshot()
    for bad in ([kids[0], kids[0]], [kids[0], root], [kids[0], 999]):
        with pytest.raises((ValueError, IndexError)):
            ctx.append_leaves(bad)
        after = ctx.snapshot()
        assert all(np.array_equal(a, b) for a, b in zip(snap[1:], after[1:]))
    with pytest.raises(ValueError):
        ctx.append_leaves(kids, [1, 0])


# ------------------------------------------------------------------ GPU
def _content_row(node, t, dim, seed):
    k, v = core.node_kv(int(node), 1, dim, seed, t0=int(t))
    return core.bf16_round(k[0]), core.bf16_round(v[0])


@pytest.mark.gpu
@pytest.mark.parametrize("use_graph,early_kv,fuse_append", [(False, 0, 1), (True, 0, 1), (True, 1, 1), (True, 0, 0)])
def test_decode_loop_matches_oracle(use_graph, early_kv, fuse_append):
    """40 decode steps of a few-shot tree (2 layers, GQA 8/2, bf16): each step
    appends one token per leaf, writes the new rows with ta_kv_append, re-plans
    and attends; outputs match the fp64 oracle on the final tree.  With
    use_graph the layer calls are one CUDA graph captured at the first step and
    replayed after every re-plan (re-captured only if graph_epoch changes).
    early_kv: CTAs load their leading KV tiles before the dependency wait,
    except tiles holding rows of the step's ta_kv_append (the last step's
    outputs depend on its appended rows).  fuse_append: the new rows are
    written inside the attention launch (default) or by ta_kv_append's own
    kernel."""
    import torch
    from gpu_helpers import dense_reference, q_tensor
    prefix, nb, steps, d, hq, hkv, n_layers = 700, 9, 40, 128, 8, 2, 2
    seeds = [11, 12]
    dim = hkv * d
    t = _few_shot(prefix, nb, 0)
    ctx = TreeAttention(n_layers=n_layers, n_q_heads=hq, n_kv_heads=hkv, d_head=d, kv_dtype="bf16",
                        max_pages=prefix // 16 + nb * (steps // 16 + 2) + 8)
    ctx.set_option("early_kv", early_kv)
    ctx.set_option("fuse_append", fuse_append)
    ctx.restore(*t.snapshot())
    for layer in range(n_layers):
        k, v = core.node_kv(0, prefix, dim, seeds[layer])
        ctx.write_kv(layer, 0, torch.from_numpy(core.bf16_round(k)).cuda().bfloat16().view(prefix, hkv, d),
                     torch.from_numpy(core.bf16_round(v)).cuda().bfloat16().view(prefix, hkv, d))
    leaves = ctx.leaves()
    L = len(leaves)
    newk = torch.empty((n_layers, L, hkv, d), dtype=torch.bfloat16, device="cuda")
    newv = torch.empty_like(newk)
    cont = [core.Content.synth(t, dim, s, qdim=hq * d).map(core.bf16_round) for s in seeds]
    qs = [q_tensor(ctx, c, leaves) for c in cont]
    outs = [torch.empty((L, hq, d), dtype=torch.float32, device="cuda") for _ in range(n_layers)]
    graph, epoch = None, None
    stream = torch.cuda.current_stream()
    for step in range(steps):
        ctx.append_leaves()
        tok = step   # the new token's index inside each branch
        for layer in range(n_layers):
            rows = [_content_row(leaf, tok, dim, seeds[layer]) for leaf in leaves]
            newk[layer].copy_(torch.from_numpy(np.stack([r[0] for r in rows]).reshape(L, hkv, d)).bfloat16())
            newv[layer].copy_(torch.from_numpy(np.stack([r[1] for r in rows]).reshape(L, hkv, d)).bfloat16())
        ctx.prepare(128, stream)
        assert ctx.kv_append_rows() == L

        def layers():
            for layer in range(n_layers):
                ctx.kv_append(layer, newk[layer], newv[layer], stream=torch.cuda.current_stream())
                ctx.attend(layer, qs[layer], outs[layer], stream=torch.cuda.current_stream())
        if not use_graph:
            layers()
        else:
            if graph is None or ctx.graph_epoch() != epoch:
                epoch = ctx.graph_epoch()
                torch.cuda.synchronize()
                # capture without executing: the step's appends must be written once
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    layers()
            graph.replay()
    torch.cuda.synchronize()
    # the decode-step fast path patched the schedule on most steps (a full
    # re-plan when a branch tail opens a new page, every 16 tokens); not with
    # early KV loads
    fast = ctx.fast_prepares()
    assert (fast == 0) if early_kv else (fast >= steps - steps // 16 - 2), fast
    snap = ctx.snapshot()
    final = core.Tree.from_snapshot(snap)
    assert final.total_tokens() == prefix + nb * steps
    for layer in range(n_layers):
        c = core.Content.synth(final, dim, seeds[layer], qdim=hq * d).map(core.bf16_round)
        ref, _ = dense_reference(snap, c, d, hq, hkv, leaves)
        got = outs[layer].cpu().numpy().astype(np.float64).reshape(L, -1)
        assert np.max(np.abs(got - ref)) <= 2e-2
        for i in range(L):
            assert core.relative_error(got[i], ref[i]) <= 1e-2, (layer, i)


@pytest.mark.gpu
def test_append_out_of_pages_is_atomic():
    """A bounded device pool: an append_leaves that does not fit fails with
    OUT_OF_MEMORY and changes nothing (no half-applied mutation)."""
    ctx = TreeAttention(n_layers=1, n_q_heads=2, n_kv_heads=2, d_head=128, kv_dtype="bf16", max_pages=4)
    root = ctx.new_tree(16)
    kids = ctx.branch(root, [16, 16])
    snap = ctx.snapshot()
    with pytest.raises(Exception):
        ctx.append_leaves()          # needs 2 pages, 1 left
    after = ctx.snapshot()
    assert all(np.array_equal(a, b) for a, b in zip(snap[1:], after[1:]))
    assert ctx.pool_stats()["page_count"] == 3
    with pytest.raises(Exception):
        ctx.branch(kids[0], [16, 16])   # 2 pages for 2 children, 1 left: rolled back
    after = ctx.snapshot()
    assert all(np.array_equal(a, b) for a, b in zip(snap[1:], after[1:]))
    ctx.append_leaves([kids[0]], [16])
    assert ctx.pool_stats()["page_count"] == 4
