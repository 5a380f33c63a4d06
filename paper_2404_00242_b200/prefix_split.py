"""Cross-GPU split of the flattened tree (the optional exchange step).

For a very long shared prefix, head sharding alone leaves each GPU streaming
the whole prefix for its heads.  Here the flattened token sequence (DFS
pre-order, the order partition_flatten streams, partition.hpp:212-253) is cut
into one contiguous range per rank instead; every rank attends ALL heads over
its range only -- its context holds the same tree topology with each node's
token count cut to the range (0-token nodes are allowed, tree.hpp) -- so every
leaf-head gets one partial (O normalised, lse) per rank.  The partials are
exchanged by head slice with one NCCL all-to-all (each rank receives its
1/world of the heads from every peer) and merged on the device in rank order
(ta_lse_merge: tree_reduce, attention.hpp:209-233).  The output is
head-sharded, as a row-parallel o_proj expects.

Traffic per layer: every rank sends (world-1)/world of L x h_q x (d + 1) fp32
(config E at 8 GPUs: 50 x 64 x 129 x 4 B x 7/8 = 1.4 MB, ~2 µs over NVLink 5);
it pays off only when the prefix work per GPU is well above that plus the
collective's latency.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .capi import check, lib


def split_counts(ids, parents, counts, n_parts):
    """Cut the flattened token sequence into n_parts contiguous ranges of
    near-equal size.  Returns, per part, an array of (offset, count) per node
    (in `ids` order): the node's tokens [offset, offset + count) that lie in
    the part's range."""
    ids = [int(x) for x in ids]
    parents = [int(x) for x in parents]
    counts = [int(x) for x in counts]
    pos = {n: i for i, n in enumerate(ids)}
    kids = {n: [] for n in ids}
    root = None
    for n, p in zip(ids, parents):
        if p < 0:
            root = n
        else:
            kids[p].append(n)   # ascending ids = insertion order (tree.hpp:207-238)
    order, stack = [], [root]
    while stack:   # DFS pre-order, children in insertion order
        n = stack.pop()
        order.append(n)
        stack.extend(reversed(kids[n]))
    total = sum(counts)
    cuts = [total * k // n_parts for k in range(n_parts + 1)]
    parts = [np.zeros((len(ids), 2), np.int64) for _ in range(n_parts)]
    start = 0
    for n in order:
        c = counts[pos[n]]
        for k in range(n_parts):
            lo, hi = max(start, cuts[k]), min(start + c, cuts[k + 1])
            if hi > lo:
                parts[k][pos[n]] = (lo - start, hi - lo)
        start += c
    return parts


def lse_merge(part_o, part_lse, out, lse_out=None, stream=None):
    """ta_lse_merge on device tensors: part_o [n][rows][d] fp32, part_lse
    [n][rows] fp32 (natural log) -> out [rows][d] (fp32 or bf16)."""
    import torch
    n, rows, d = part_o.shape
    for t in (part_o, part_lse, out):
        if not t.is_contiguous() or t.device.type != "cuda":
            raise ValueError("lse_merge: contiguous CUDA tensors expected")
    if part_o.dtype != torch.float32 or part_lse.dtype != torch.float32 or tuple(part_lse.shape) != (n, rows):
        raise ValueError("lse_merge: part_o [n][rows][d] and part_lse [n][rows] fp32 expected")
    if out.numel() != rows * d or out.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("lse_merge: out [rows][d] fp32 or bf16 expected")
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib().ta_lse_merge(C.c_void_p(part_o.data_ptr()), C.c_void_p(part_lse.data_ptr()), n, rows, d,
                             C.c_void_p(out.data_ptr()), int(out.dtype == torch.bfloat16),
                             C.c_void_p(lse_out.data_ptr() if lse_out is not None else 0), C.c_void_p(s)),
          "lse_merge")
    return out


def exchange_by_heads(out_r, lse_r, world, group=None):
    """All-to-all of one rank's partials by head slice: out_r [L][h][d] fp32,
    lse_r [L][h] -> (recv_o [world][L * h/world][d], recv_lse [world][L * h/world]),
    part k = rank k's partial for this rank's heads.  One NCCL all_to_all_single
    per tensor (gloo on CPU)."""
    import torch
    import torch.distributed as dist
    L, h, d = out_r.shape
    hs = h // world
    send_o = out_r.view(L, world, hs, d).permute(1, 0, 2, 3).contiguous()
    send_l = lse_r.view(L, world, hs).permute(1, 0, 2).contiguous()
    recv_o = torch.empty_like(send_o)
    recv_l = torch.empty_like(send_l)
    dist.all_to_all_single(recv_o, send_o, group=group)
    dist.all_to_all_single(recv_l, send_l, group=group)
    return recv_o.view(world, L * hs, d), recv_l.view(world, L * hs)


class PrefixSplitAttention:
    """One rank of the split: a TreeAttention context over this rank's token
    range with all heads, plus the exchange and merge.  q is the full
    [L][h_q][d]; attend() returns this rank's head slice [L][h_q / world][d]."""

    def __init__(self, snapshot, rank, world, group=None, **ctx_kwargs):
        from .api import TreeAttention
        root, ids, parents, counts = snapshot
        self.rank, self.world, self.group = rank, world, group
        self.ranges = split_counts(ids, parents, counts, world)[rank]
        self.ids = [int(x) for x in ids]
        self.ctx = TreeAttention(**{**ctx_kwargs, "out_dtype": "f32"})   # partials in fp32
        self.ctx.restore(root, ids, parents, [int(c) for _, c in self.ranges])
        if self.ctx.n_local_q_heads % world:
            raise ValueError("prefix split: q heads must divide across ranks")

    def write_kv(self, layer, node, k, v):
        """k, v: the node's FULL KV [n_tok][h_kv][d]; this rank keeps its range."""
        off, cnt = (int(x) for x in self.ranges[self.ids.index(int(node))])
        if cnt:
            self.ctx.write_kv(layer, int(node), k[off:off + cnt].contiguous(), v[off:off + cnt].contiguous())

    def attend(self, layer, q, out=None, stream=None):
        import torch
        L, hq, d = q.shape
        o_r = torch.empty((L, hq, d), dtype=torch.float32, device=q.device)
        l_r = torch.empty((L, hq), dtype=torch.float32, device=q.device)
        self.ctx.attend(layer, q, o_r, lse=l_r, stream=stream)
        recv_o, recv_l = exchange_by_heads(o_r, l_r, self.world, self.group)
        if out is None:
            out = torch.empty((L, hq // self.world, d), dtype=q.dtype, device=q.device)
        return lse_merge(recv_o, recv_l, out.view(-1, d), stream=stream).view(L, hq // self.world, d)
