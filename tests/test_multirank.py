"""Head sharding over ranks, on CPU with the gloo backend.

Each rank builds a host-only context owning kv heads
[rank*h_kv/N, (rank+1)*h_kv/N) -- exactly what bench.py does per GPU under
torchrun.  The plan and the lane/tile structure are head-independent and
must be identical on every rank; each rank's fp64 interpretation of its own
schedule, all-gathered, must equal the unsharded oracle (no collective is
needed on the attention path: outputs are head-disjoint)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import core


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
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from test_schedule import interpret
        from paper_2404_00242_b200 import TreeAttention

        h_kv, G, d = 4, 2, 16
        n_loc = h_kv // world
        rng = core.Rng(4242)
        t = core.random_tree(rng, max_leaves=24, max_tokens=1500, max_node_tokens=120)
        snap = t.snapshot()
        ctx = TreeAttention(device=-1, n_q_heads=h_kv * G, n_kv_heads=h_kv, d_head=d, kv_dtype="f32",
                            kv_head_begin=rank * n_loc, n_local_kv_heads=n_loc)
        ctx.set_option("num_ctas", 11)
        ctx.restore(*snap)
        S = ctx.schedule(64)
        # head-independent structure: identical on all ranks
        sig = torch.tensor([S["n_lanes"], len(S["tile_ng"]), int(S["grp_row"].sum()), int(S["grp_info"].sum()),
                            len(ctx.plan_json(64))], dtype=torch.int64)
        sigs = [torch.zeros_like(sig) for _ in range(world)]
        dist.all_gather(sigs, sig)
        assert all(torch.equal(x, sigs[0]) for x in sigs)
        assert set(int(h) for h in S["items"][:, 0]) == set(range(n_loc))
        # each rank: its kv heads' outputs (fp64 schedule interpretation, one head at a time)
        c = core.Content.synth(t, h_kv * d, 7, qdim=h_kv * G * d)
        L = len(t.leaves())
        mine = np.zeros((L, n_loc * G * d))
        one = TreeAttention(device=-1, n_q_heads=G, n_kv_heads=1, d_head=d, kv_dtype="f32")
        one.set_option("num_ctas", 11)
        one.restore(*snap)
        for hl in range(n_loc):
            h = rank * n_loc + hl
            ch = core.Content(
                {n: k[:, h * d:(h + 1) * d] for n, k in c.keys.items()},
                {n: v[:, h * d:(h + 1) * d] for n, v in c.values.items()},
                {n: q[h * G * d:(h + 1) * G * d] for n, q in c.queries.items()}, d)
            mine[:, hl * G * d:(hl + 1) * G * d] = interpret(one, t, ch, d, G, 1, 64)
        parts = [torch.zeros(L, n_loc * G * d, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        if rank == 0:
            full = torch.cat(parts, dim=1).numpy()
            ref = core.naive_attention(t, c.expanded(d, h_kv * G, h_kv), d, h_kv * G)
            for i, leaf in enumerate(t.leaves()):
                if t.path_tokens(int(leaf)) > 0:
                    assert core.relative_error(full[i], ref[i]) < 1e-12, i
            open(os.path.join(result_dir, "ok"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_head_sharded_two_ranks_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert (tmp_path / "ok").exists()
