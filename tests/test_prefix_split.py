"""Cross-GPU prefix split (paper_2404_00242_b200/prefix_split.py).

* split_counts cuts the flattened (DFS pre-order) token sequence into
  contiguous, near-equal ranges covering every token exactly once.
* gloo, world_size 2 (CPU): each rank's partial over its range for ALL heads
  (fp64 restatement of group_attention, attention.hpp:117-204 -- the CUDA
  kernel's stand-in), exchanged by head slice with the product's
  exchange_by_heads (all_to_all_single) and merged by tree_reduce
  (attention.hpp:209-233), equals naive_attention for the rank's heads.
* GPU (one device, ranks simulated): per-range contexts through the tcgen05
  kernel, the same exchange as local slicing, and the product's ta_lse_merge
  kernel, against the dense fp64 reference (bf16 gates)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import core
from paper_2404_00242_b200.prefix_split import exchange_by_heads, split_counts


def _path(t, leaf):
    out, cur = [], int(leaf)
    while cur != -1:
        out.append(cur)
        cur = t.parent(cur)
    return out[::-1]


def test_split_counts_cover_once():
    rng = core.Rng(31)
    for trial in range(30):
        t = core.random_tree(rng, max_leaves=20, max_tokens=3000, max_node_tokens=400)
        root, ids, par, cnt = t.snapshot()
        total = int(sum(cnt))
        for n in (1, 2, 3, 5, 8):
            parts = split_counts(ids, par, cnt, n)
            got = np.zeros(len(ids), np.int64)
            sizes = []
            for p in parts:
                got += p[:, 1]
                sizes.append(int(p[:, 1].sum()))
                for i, (off, c) in enumerate(p):
                    assert 0 <= off and off + c <= int(cnt[i])
            assert np.array_equal(got, np.asarray(cnt, np.int64))
            assert max(sizes) - min(sizes) <= 1 and sum(sizes) == total


def _partial(t, c, ranges, ids, d, h_q, h_kv):
    """fp64 attention of every leaf over the tokens of its path inside `ranges`
    (node -> (offset, count)): (out [L][h_q][d], lse [L][h_q], natural log)."""
    G = h_q // h_kv
    pos = {int(n): i for i, n in enumerate(ids)}
    leaves = list(t.leaves())
    out = np.zeros((len(leaves), h_q, d))
    lse = np.full((len(leaves), h_q), -np.inf)
    for li, leaf in enumerate(leaves):
        K, V = [], []
        for n in _path(t, leaf):
            off, cnt = (int(x) for x in ranges[pos[n]])
            if cnt:
                K.append(c.keys[n][off:off + cnt])
                V.append(c.values[n][off:off + cnt])
        if not K:
            continue
        K = np.concatenate(K).astype(np.float64).reshape(-1, h_kv, d)
        V = np.concatenate(V).astype(np.float64).reshape(-1, h_kv, d)
        q = c.queries[int(leaf)].astype(np.float64).reshape(h_q, d)
        hk = np.arange(h_q) // G
        s = np.einsum("thd,hd->ht", K[:, hk], q) / np.sqrt(d)
        m = s.max(1, keepdims=True)
        w = np.exp(s - m)
        out[li] = np.einsum("ht,thd->hd", w / w.sum(1, keepdims=True), V[:, hk])
        lse[li] = (m + np.log(w.sum(1, keepdims=True))).ravel()
    return out, lse


def _tree_reduce(parts_o, parts_l):
    """tree_reduce over parts (attention.hpp:209-233): [n][rows][d], [n][rows]."""
    M = parts_l.max(0)
    w = np.where(np.isfinite(parts_l), np.exp(parts_l - np.where(np.isfinite(M), M, 0)), 0.0)
    den = w.sum(0)
    return (w[..., None] * parts_o).sum(0) / np.where(den > 0, den, 1)[:, None]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h_kv, G, d = 2, 4, 16
        h_q = h_kv * G
        t = core.Tree(700)                     # one long shared prefix ...
        kids = t.branch(t.root, [40, 0, 90])   # ... and branches (one empty)
        t.branch(kids[0], [15, 25])
        root, ids, par, cnt = t.snapshot()
        c = core.Content.synth(t, h_kv * d, 11, qdim=h_q * d)
        ranges = split_counts(ids, par, cnt, world)[rank]
        o_r, l_r = _partial(t, c, ranges, ids, d, h_q, h_kv)
        L = o_r.shape[0]
        recv_o, recv_l = exchange_by_heads(torch.from_numpy(o_r), torch.from_numpy(l_r), world)
        mine = _tree_reduce(recv_o.numpy(), recv_l.numpy()).reshape(L, h_q // world, d)
        ref = core.naive_attention(t, c.expanded(d, h_q, h_kv), d, h_q).reshape(L, h_q, d)
        hs = h_q // world
        for i, leaf in enumerate(t.leaves()):
            if t.path_tokens(int(leaf)) > 0:
                assert core.relative_error(mine[i].ravel(), ref[i, rank * hs:(rank + 1) * hs].ravel()) < 1e-12
        open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_prefix_split_two_ranks_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_prefix_split_kernels_one_device(world):
    """Ranks simulated on cuda:0: per-range tcgen05 partials (all 8 kv heads),
    the all-to-all as slicing, ta_lse_merge -> each rank's head slice."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from gpu_helpers import dense_reference, make_content
    from paper_2404_00242_b200 import TreeAttention
    from paper_2404_00242_b200.prefix_split import lse_merge
    h_q, h_kv, d = 32, 8, 128
    t = core.Tree(6000)
    t.branch(t.root, [300] * 12)
    snap = t.snapshot()
    root, ids, par, cnt = snap
    c = make_content(t, d, h_q, h_kv, 5, bf16=True)
    parts = split_counts(ids, par, cnt, world)
    L = len(t.leaves())
    outs, lses = [], []
    for r in range(world):
        ctx = TreeAttention(n_layers=1, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype="bf16", out_dtype="f32",
                            max_pages=int(sum((int(x) + 15) // 16 for x in cnt)) + 16, device=0)
        ctx.restore(root, ids, par, [int(x) for x in parts[r][:, 1]])
        for i, n in enumerate(ids):
            off, cn = (int(x) for x in parts[r][i])
            if cn:
                k = torch.from_numpy(c.keys[int(n)][off:off + cn].reshape(cn, h_kv, d)).bfloat16().cuda()
                v = torch.from_numpy(c.values[int(n)][off:off + cn].reshape(cn, h_kv, d)).bfloat16().cuda()
                ctx.write_kv(0, int(n), k, v)
        q = torch.from_numpy(np.stack([c.queries[int(lf)] for lf in ctx.leaves()]).reshape(L, h_q, d)).bfloat16().cuda()
        lse = torch.empty((L, h_q), device="cuda")
        ctx.prepare(128)
        outs.append(ctx.attend(0, q, lse=lse).float())
        lses.append(lse)
    ref, _ = dense_reference(snap, c, d, h_q, h_kv, t.leaves())
    ref = ref.reshape(L, h_q, d)
    hs = h_q // world
    for r in range(world):   # what rank r receives: every rank's partial for its heads
        po = torch.stack([o[:, r * hs:(r + 1) * hs] for o in outs]).reshape(world, L * hs, d).contiguous()
        pl = torch.stack([x[:, r * hs:(r + 1) * hs] for x in lses]).reshape(world, L * hs).contiguous()
        got = lse_merge(po, pl, torch.empty((L * hs, d), device="cuda")).view(L, hs, d).cpu().numpy()
        want = ref[:, r * hs:(r + 1) * hs]
        assert np.abs(got - want).max() <= 2e-2
        assert max(core.relative_error(got[i].ravel(), want[i].ravel()) for i in range(L)) <= 1e-2
