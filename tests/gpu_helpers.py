"""Shared helpers for the GPU parity tests, smoke() and bench.py: load a tree
and its content into a TreeAttention context and compare with the oracle.

The checker side (oracle.core, np_reference) is test infrastructure; the
product side is only ever reached through paper_2404_00242_b200 (C ABI)."""
from __future__ import annotations

import numpy as np

from oracle import core


def np_reference(snap, content: core.Content, d_head: int, h_q: int, h_kv: int, leaves=None, leaf_idx=None):
    """fp64 attention over each leaf's root-to-leaf KV with GQA head mapping
    (q head h reads kv head h // (h_q/h_kv)) -- the same math as
    naive_attention (attention.hpp:237-288), vectorised.  Returns
    (out [n][h_q*d], lse [n][h_q]) for the selected leaf indices."""
    root, ids, par, cnt = snap
    parent = {int(i): int(p) for i, p in zip(ids, par)}
    G = h_q // h_kv
    if leaf_idx is None:
        leaf_idx = range(len(leaves))
    outs, lses = [], []
    for li in leaf_idx:
        leaf = int(leaves[li])
        chain = []
        cur = leaf
        while cur != -1:
            chain.append(cur)
            cur = parent[cur]
        chain.reverse()
        K = np.concatenate([content.keys[n] for n in chain]).astype(np.float64)
        V = np.concatenate([content.values[n] for n in chain]).astype(np.float64)
        q = content.queries[leaf].astype(np.float64).reshape(h_q, d_head)
        T = K.shape[0]
        if T == 0:
            outs.append(np.zeros(h_q * d_head))
            lses.append(np.full(h_q, -np.inf))
            continue
        K = K.reshape(T, h_kv, d_head)
        V = V.reshape(T, h_kv, d_head)
        Kq = K[:, np.arange(h_q) // G, :]                      # [T][h_q][d]
        Vq = V[:, np.arange(h_q) // G, :]
        s = np.einsum("thd,hd->ht", Kq, q) / np.sqrt(d_head)  # [h_q][T]
        m = s.max(axis=1, keepdims=True)
        w = np.exp(s - m)
        den = w.sum(axis=1, keepdims=True)
        o = np.einsum("ht,thd->hd", w / den, Vq)
        outs.append(o.reshape(-1))
        lses.append((m + np.log(den)).ravel())
    return np.array(outs), np.array(lses)


def make_content(tree: core.Tree, d_head: int, h_q: int, h_kv: int, seed: int, bf16: bool, q_scale: float = 1.0):
    """Reference content (fill_tree_kv / make_queries, synth.hpp:41-69): K/V at
    h_kv*d, queries at h_q*d; bf16 rounds every input."""
    c = core.Content.synth(tree, h_kv * d_head, seed, qdim=h_q * d_head)
    if q_scale != 1.0:
        c.queries = {k: (v * np.float32(q_scale)).astype(np.float32) for k, v in c.queries.items()}
    if bf16:
        c = c.map(core.bf16_round)
    return c


def load_into(ctx, content: core.Content, layer: int = 0, kv_head_begin: int = 0):
    """PagePool::write_kv for every node (device-side source)."""
    import torch
    dt = torch.bfloat16 if ctx.kv_dtype == "bf16" else torch.float32
    nl, d = ctx.n_local_kv_heads, ctx.d_head
    for node, K in content.keys.items():
        n = K.shape[0]
        if n == 0:
            continue
        sl = slice(kv_head_begin * d, (kv_head_begin + nl) * d)
        k = torch.from_numpy(np.ascontiguousarray(K[:, sl])).to("cuda").to(dt).reshape(n, nl, d)
        v = torch.from_numpy(np.ascontiguousarray(content.values[node][:, sl])).to("cuda").to(dt).reshape(n, nl, d)
        ctx.write_kv(layer, node, k, v)


def q_tensor(ctx, content: core.Content, leaves, q_head_begin: int = 0):
    import torch
    dt = torch.bfloat16 if ctx.kv_dtype == "bf16" else torch.float32
    d, hl = ctx.d_head, ctx.n_local_q_heads
    Q = np.stack([content.queries[int(l)] for l in leaves]).reshape(len(leaves), -1, d)
    Q = Q[:, q_head_begin:q_head_begin + hl, :]
    return torch.from_numpy(np.ascontiguousarray(Q)).to("cuda").to(dt)


def run_gpu(snap, content: core.Content, d_head: int, h_q: int, h_kv: int, kv_dtype: str = "f32",
            block_size: int = 128, options: dict | None = None, out_dtype: str = "f32", with_lse: bool = False):
    """Tree + content -> TreeAttention (1 layer) -> (out [L][h_q*d] fp64, lse, ctx)."""
    import torch
    from paper_2404_00242_b200 import TreeAttention
    root, ids, par, cnt = snap
    pages = int(sum((int(c) + 15) // 16 for c in cnt)) + 8
    ctx = TreeAttention(n_layers=1, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d_head, kv_dtype=kv_dtype,
                        out_dtype=out_dtype, max_pages=pages, device=0)
    for k, v in (options or {}).items():
        ctx.set_option(k, v)
    ctx.restore(*snap)
    load_into(ctx, content)
    leaves = ctx.leaves()
    q = q_tensor(ctx, content, leaves)
    lse = torch.full((len(leaves), h_q), float("nan"), device="cuda") if with_lse else None
    ctx.prepare(block_size)
    out = ctx.attend(0, q, lse=lse)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy().astype(np.float64).reshape(len(leaves), -1)
    return o, (lse.cpu().numpy() if with_lse else None), ctx


def dense_reference(snap, content: core.Content, d_head: int, h_q: int, h_kv: int, leaves, kv_heads=None):
    """fp64 reference for full-size trees: the dense form of naive_attention
    (attention.hpp:237-288) with the tree mask written as the ancestor relation
    (reconstruct_dense_mask, partition.hpp:267-279): leaf l attends token t iff
    t's node lies on l's root-to-leaf path.  One BLAS GEMM per kv head.
    `content` holds K/V for the kv heads in `kv_heads` (default: all) side by
    side and queries for their G q heads each.  Returns (out [L][hq*d], lse
    [L][hq]) for the selected heads, in leaves() order."""
    root, ids, par, cnt = snap
    parent = {int(i): int(p) for i, p in zip(ids, par)}
    kv_heads = list(range(h_kv)) if kv_heads is None else list(kv_heads)
    G = h_q // h_kv
    nodes = [int(i) for i, c in zip(ids, cnt) if int(c) > 0]
    tok_node = np.concatenate([np.full(int(content.keys[n].shape[0]), n, np.int64) for n in nodes]) \
        if nodes else np.zeros(0, np.int64)
    K = np.concatenate([content.keys[n] for n in nodes]) if nodes else np.zeros((0, len(kv_heads) * d_head))
    V = np.concatenate([content.values[n] for n in nodes]) if nodes else np.zeros((0, len(kv_heads) * d_head))
    L = len(leaves)
    mask = np.zeros((L, tok_node.size), bool)
    for li, leaf in enumerate(leaves):
        path = []
        cur = int(leaf)
        while cur != -1:
            path.append(cur)
            cur = parent[cur]
        mask[li] = np.isin(tok_node, path)
    Q = np.stack([content.queries[int(l)] for l in leaves]).astype(np.float64).reshape(L, len(kv_heads) * G, d_head)
    out = np.zeros((L, len(kv_heads) * G, d_head))
    lse = np.full((L, len(kv_heads) * G), -np.inf)
    big = np.repeat(mask, G, axis=0)   # [L*G][N]
    for hi in range(len(kv_heads)):
        Kh = K[:, hi * d_head:(hi + 1) * d_head].astype(np.float64)
        Vh = V[:, hi * d_head:(hi + 1) * d_head].astype(np.float64)
        q = Q[:, hi * G:(hi + 1) * G, :].reshape(L * G, d_head)
        s = (q @ Kh.T) / np.sqrt(d_head)
        s[~big] = -np.inf
        m = s.max(axis=1, keepdims=True)
        ok = np.isfinite(m[:, 0])
        m[~ok] = 0.0
        w = np.exp(s - m)
        den = w.sum(axis=1, keepdims=True)
        o = (w @ Vh) / np.where(den > 0, den, 1.0)
        out[:, hi * G:(hi + 1) * G, :] = o.reshape(L, G, d_head)
        l_ = np.where(ok, m[:, 0] + np.log(np.where(den[:, 0] > 0, den[:, 0], 1.0)), -np.inf)
        lse[:, hi * G:(hi + 1) * G] = l_.reshape(L, G)
    return out.reshape(L, -1), lse
