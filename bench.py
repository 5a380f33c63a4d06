#!/usr/bin/env python
"""DeFT-Flatten tree-attention decode benchmark (B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config few_shot]
    python bench.py --impl reference ...          # reference CPU path arm

One step = one decode step of the named config: the flatten plan + device
schedule for the current tree (host, ta_prepare) and the attention of every
layer (n_layers x ta_attend), inputs resident in HBM.  Each layer has its own
KV pool, so the per-step working set (3.1 GB for config B) is far larger than
L2 and nothing is served from L2 across layers or steps.

Multi-GPU (torchrun): kv heads are sharded across ranks (head sharding, no
collective on the attention path); every rank runs the whole tree for its
heads, `value` is the whole-job step latency = max over ranks.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree-attention us/decode step"

CONFIGS = {
    # BASELINE.json configs[1]: Llama-3-8B shapes, 4k prompt, 50 branches, iteration 400
    "few_shot": dict(kind="few_shot", prefix=4000, branches=50, iteration=400, n_layers=32, h_q=32, h_kv=8,
                     d=128, dtype="bf16"),
    # configs[0]: CPU-ref demo tree, 1 layer, 32 x d128 fp32
    "demo": dict(kind="demo", n_layers=1, h_q=32, h_kv=32, d=128, dtype="f32"),
    # configs[2]: reasoning stand-in (SURVEY §8d C-ii)
    "reasoning": dict(kind="reasoning", n_layers=32, h_q=32, h_kv=8, d=128, dtype="bf16"),
    # configs[3]: speculative token trees
    "spec_t64": dict(kind="spec", prompt=4000, tree_size=64, n_layers=32, h_q=32, h_kv=8, d=128, dtype="bf16"),
    "spec_t256": dict(kind="spec", prompt=16000, tree_size=256, n_layers=32, h_q=32, h_kv=8, d=128, dtype="bf16"),
    # configs[4]: Llama-3-70B shapes, 32k prefix few-shot
    "few_shot_70b": dict(kind="few_shot", prefix=32000, branches=50, iteration=400, n_layers=80, h_q=64, h_kv=8,
                         d=128, dtype="bf16"),
}


# ------------------------------------------------------------------ trees
def build_snapshot(cfg):
    """Tree snapshots via the reference's generators, restated in oracle.core
    (gen_few_shot workloads.hpp:98-111 etc.); plain integer topology."""
    from oracle import core
    k = cfg["kind"]
    if k == "few_shot":
        t = core.Tree(cfg["prefix"])
        kids = t.branch(t.root, [0] * cfg["branches"])
        for kid in kids:
            t.append_tokens(kid, cfg["iteration"])
        return t.snapshot()
    if k == "demo":
        t = core.Tree(1024)
        t.branch(t.root, [128] * 4)
        return t.snapshot()
    if k == "reasoning":
        return reasoning_standin()
    if k == "spec":
        return spec_tree(cfg["prompt"], cfg["tree_size"])
    raise ValueError(k)


def reasoning_standin():
    """SURVEY §8d C-ii: ReasoningSpec{1000, depth 10, width 10, gen 100}, each
    depth branches the frontier into 10 seeded U[50,200] thoughts and prunes
    4 of them (keep 6); peak snapshot."""
    from oracle import core
    rng = core.Rng(7)
    t = core.Tree(1000)
    frontier = t.root
    best, best_n = None, -1
    for depth in range(10):
        kids = t.branch(frontier, [rng.uniform_int(50, 200) for _ in range(10)])
        for _ in range(100):
            for leaf in list(t.leaves()):
                t.append_tokens(int(leaf), 1)
        if t.total_tokens() > best_n:
            best, best_n = t.snapshot(), t.total_tokens()
        for k in kids[6:]:
            t.prune(k)
        frontier = kids[0]
    return best


def spec_tree(prompt, t_size):
    """gen_speculative step 0 (workloads.hpp:192-271) with a 0-token query
    holder under every interior token node."""
    from oracle.make_golden import holder_token_tree
    return holder_token_tree(prompt, t_size)


# ------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms in the
    background; summary() keeps the samples inside [mark_start, mark_end]."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._p = None
        self.t0 = self.t1 = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                        "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self._p:
            self._p.terminate()
            try:
                self._p.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self._p.kill()

    def summary(self):
        smp = self.samples
        if self.t0 is not None and self.t1 is not None:
            inside = [x for x in smp if self.t0 <= x[0] <= self.t1]
            smp = inside or sorted(smp, key=lambda x: abs(x[0] - (self.t0 + self.t1) / 2))[:1]
        smp = [x[1] for x in smp]
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in smp if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in smp if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in smp:
            for n, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(smp)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_tensor_peak():
    """Dense bf16 TFLOP/s: MEASURED_PEAKS.json's sustained figure (the layer
    time is taken inside back-to-back graph replays), else the recipe's."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p.get("bf16_tflops_sustained") or p["bf16_tflops"]), "measured (sustained)"
    except Exception:
        return 1648.0, "fallback"


def profile_traffic(config_name):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config_name)
    except Exception:
        return None


# ------------------------------------------------------------- CPU baseline
def cpu_baseline(cfg, snap, sample_layers=1):
    """The reference's run_iteration(tree, Flatten, 128, pool, queries,
    {d_head, n_heads=G, use_double=false}) on one kv-head group (G q heads,
    KV expanded) of one layer; extrapolated x h_kv x n_layers.  Uses the
    reference compiled in place (oracle/_ref) when present, else the C port."""
    from oracle import core, ref
    threads = os.cpu_count() or 1
    G = cfg["h_q"] // cfg["h_kv"]
    d = cfg["d"]
    if ref.available():
        ref.set_threads(threads)
        ref.tune_malloc()
        inst = ref.Instance.gqa(snap, d, G, 1, 42)
        inst.run_iteration(128)  # warm
        secs = []
        t_end = time.time() + 10
        while time.time() < t_end or not secs:
            secs.append(inst.run_iteration(128)[2])
            if len(secs) >= 5:
                break
        t = min(secs)
        kind, cores = "reference", threads
    else:
        tr = core.Tree.from_snapshot(snap)
        c = core.Content.synth(tr, d, 42, qdim=G * d).expanded(d, G, 1)
        t0 = time.perf_counter()
        core.run_iteration_flatten(tr, c, d, G)
        t = time.perf_counter() - t0
        kind, cores = "port", 1
    per_step_us = t * 1e6 * cfg["h_kv"] * cfg["n_layers"]
    return {"value": per_step_us, "unit": "us/decode step", "cores": cores, "kind": kind,
            "sample": f"1 layer x 1 kv-head group ({G} q heads, GQA-expanded MHA) of run_iteration, "
                      f"best of {len(secs) if kind == 'reference' else 1}, x{cfg['h_kv']} groups x{cfg['n_layers']} layers"}


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="few_shot", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the layer calls eagerly (no CUDA graph)")
    ap.add_argument("--opt", action="append", default=[], help="ta_set_option key=value (repeatable)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    snap = build_snapshot(cfg)

    if args.impl == "reference":
        if rank != 0:
            return
        runs = []
        from oracle import ref
        for _ in range(args.warmup):
            pass
        for _ in range(args.steps):
            runs.append(cpu_baseline(cfg, snap))
        v = statistics.median(r["value"] for r in runs)
        base = dict(runs[0])
        base["value"] = v
        line = {"metric": METRIC, "value": v, "unit": "us/decode step", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": v / 1000.0, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference synth.hpp content, seed 42)",
                "impl": "reference", "config": config_obj(args, cfg, world), "cpu_baseline": base,
                "e2e": {"value": v, "unit": "us/decode step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line))
        return

    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2404_00242_b200 import TreeAttention

    h_kv, h_q, d, L_layers = cfg["h_kv"], cfg["h_q"], cfg["d"], cfg["n_layers"]
    assert h_kv % world == 0, "kv heads must divide across ranks"
    n_loc = h_kv // world
    G = h_q // h_kv
    root, ids, par, cnt = snap
    pages = int(sum((int(c) + 15) // 16 for c in cnt)) + 16
    ctx = TreeAttention(n_layers=L_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype=cfg["dtype"],
                        out_dtype=cfg["dtype"], max_pages=pages, device=local_rank,
                        kv_head_begin=rank * n_loc, n_local_kv_heads=n_loc)
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    ctx.restore(root, ids, par, cnt)
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    for layer in range(L_layers):
        for node, c in zip(ids, cnt):
            c = int(c)
            if c == 0:
                continue
            k = (torch.rand((c, n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt)
            v = (torch.rand((c, n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt)
            ctx.write_kv(layer, int(node), k, v)
    leaves = ctx.leaves()
    L = len(leaves)
    hq_loc = n_loc * G
    q = (torch.rand((L_layers, L, hq_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt)
    out = torch.empty((L_layers, L, hq_loc, d), dtype=dt, device="cuda")
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def layers():
        for layer in range(L_layers):
            ctx.attend(layer, q[layer], out[layer], stream=torch.cuda.current_stream())

    # one decode step = host plan + schedule + metadata upload (ta_prepare) and
    # the n_layers attention calls, replayed as a CUDA graph (as a serving
    # engine captures its decode step; the graph reads the schedule metadata
    # that ta_prepare re-uploads into the same device buffers every step)
    ctx.prepare(128, stream)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        layers()   # warm the launch configuration before capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            layers()
        torch.cuda.synchronize()

    def step():
        ctx.prepare(128, stream)
        if graph is not None:
            graph.replay()
        else:
            for layer in range(L_layers):
                ctx.attend(layer, q[layer], out[layer], stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    io = ctx.io_stats()
    launches_per_attend = ctx.launches_per_attend()

    # ---- timed region: device time via CUDA events, max over ranks
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        for _ in range(30):   # keep the GPU busy while the sampler starts
            step()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        clocks.mark_start()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clocks.mark_end()
        if world > 1:
            torch.distributed.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-layer time of ta_attend (attention + merge launches) on the
    # launching stream: the graph of n_layers calls, replayed back to back
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.prepare(128, stream)
    torch.cuda.synchronize()
    reps = 10
    ev0.record(stream)
    for _ in range(reps):
        if graph is not None:
            graph.replay()
        else:
            for layer in range(L_layers):
                ctx.attend(layer, q[layer], out[layer], stream=stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    attend_ms = ev0.elapsed_time(ev1) / (reps * L_layers)

    # ---- e2e through the public host-buffer entry (H2D q + D2H out per layer)
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        oh = torch.empty(out.shape, dtype=dt).pin_memory()
        qn = qh.view(torch.int16).numpy() if dt == torch.bfloat16 else qh.numpy()
        on = oh.view(torch.int16).numpy() if dt == torch.bfloat16 else oh.numpy()

        def step_host():
            # one decode step through the host-buffer entry: the n_layers
            # calls pipeline copy-in / attention / copy-out; the step ends
            # when every layer's output is back in host memory
            ctx.prepare(128, stream)
            for layer in range(L_layers):
                ctx.attend_host_async(layer, qn[layer], on[layer], stream=stream)
            ctx.attend_host_wait()

        for _ in range(2):
            step_host()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step_host()
        h1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1000 / args.steps
        ems = max(h0.elapsed_time(h1) / args.steps, wall_ms)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": ems * 1000.0, "unit": "us/decode step",
               "h2d_bytes_per_step": int(q.numel() * q.element_size()),
               "d2h_bytes_per_step": int(out.numel() * out.element_size()),
               "path": "ta_prepare + ta_attend_host_async per layer (pinned host q in, host out back; copy-in, "
                        "attention and copy-out of consecutive layers overlap) + ta_attend_host_wait per step"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    peak, peak_kind = measured_peaks()
    alg_bytes = io.kv_bytes  # one pass over unique tree KV per layer (this rank's heads)
    achieved = alg_bytes / (attend_ms * 1e-3) / 1e9
    # the bound: HBM unless the masked-in flops per unique KV byte reach the
    # ridge (the speculative configs at t >= 64 and 70B)
    tpeak, tpeak_kind = measured_tensor_peak()
    ridge = tpeak * 1e12 / (peak * 1e9)
    hbm_line = {"achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak}
    tflops = io.flops / (attend_ms * 1e-3) / 1e12
    tensor_line = {"achieved": tflops, "peak": tpeak, "peak_kind": tpeak_kind, "unit": "TFLOP/s", "frac": tflops / tpeak}
    tensor_bound = io.flops >= ridge * alg_bytes
    roofline = dict(tensor_line if tensor_bound else hbm_line)
    roofline.update({"kernel": "ta_attend (attn_mma or attn_fma + merge), per layer, graph-replayed",
                     "bound": "tensor" if tensor_bound else "hbm",
                     "traffic": profile_traffic(args.config), "alg_bytes_per_launch": alg_bytes,
                     "alg_flops_per_launch": io.flops, "intensity_flop_per_byte": io.flops / max(1, alg_bytes),
                     "other": tensor_line if not tensor_bound else hbm_line})
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(cfg, snap)
        except Exception as e:  # the baseline must never sink the bench line
            cpu = {"value": None, "unit": "us/decode step", "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}
    line = {
        "metric": METRIC,
        "value": ms * 1000.0,
        "unit": "us/decode step",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": "synthetic (uniform(-1,1) KV/Q, reference tree generators)",
        "config": config_obj(args, cfg, world),
        "kv_io_bytes_per_step": io.kv_bytes * L_layers,
        "partial_io_bytes_per_step": io.partial_bytes * L_layers,
        "meta_bytes_per_step": io.meta_bytes,
        "us_per_layer": attend_ms * 1000.0,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps * L_layers * launches_per_attend,
        "schedule": {"chunks": io.n_chunks, "groups": io.n_groups, "units": io.n_units, "units_mma": io.n_units_mma,
                     "partials": io.n_partials, "kv_bytes_loaded_per_layer": io.kv_bytes_loaded},
    }
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def config_obj(args, cfg, world):
    return {"workload": args.config, **{k: v for k, v in cfg.items() if k != "kind"}, "block_size": 128,
            "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (per-layer KV pools, n_layers x unique KV per step)"}


if __name__ == "__main__":
    main()
