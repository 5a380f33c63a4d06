#!/usr/bin/env python
"""DeFT-Flatten tree-attention decode benchmark (B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config few_shot]
    python bench.py --impl reference ...          # reference CPU path arm

One step = one decode step of the named config: the flatten plan + device
schedule for the current tree (host, ta_prepare) and the attention of every
layer (n_layers x ta_attend), inputs resident in HBM.  Each layer has its own
KV pool, so the per-step working set (3.1 GB for config B) is far larger than
L2 and nothing is served from L2 across layers or steps.

The headline line is config B (few-shot, BASELINE.json configs[1]).  At N = 1
the default run also measures the other benchmarked configs (C reasoning, D
speculative t64 / t256, E's per-GPU shard) and reports them under "configs"
with their own roofline, e2e and CPU baseline (--headline-only skips them).

Multi-GPU (torchrun): kv heads are sharded across ranks (head sharding, no
collective on the attention path); every rank runs the whole tree for its
heads, `value` is the whole-job step latency = max over ranks.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
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
    # configs[4]: Llama-3-70B shapes, 32k prefix few-shot: all 8 kv heads on one GPU ...
    "few_shot_70b": dict(kind="few_shot", prefix=32000, branches=50, iteration=400, n_layers=80, h_q=64, h_kv=8,
                         d=128, dtype="bf16"),
    # ... and the per-GPU shard of the 8-GPU head-sharded run (1 kv head + its 8 q heads)
    "few_shot_70b_shard": dict(kind="few_shot", prefix=32000, branches=50, iteration=400, n_layers=80, h_q=64,
                               h_kv=8, n_local_kv_heads=1, d=128, dtype="bf16"),
}
SUB_CONFIGS = ["reasoning", "spec_t64", "spec_t256", "few_shot_70b_shard"]


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


def local_kv_heads(cfg, world):
    return cfg.get("n_local_kv_heads") or cfg["h_kv"] // world


# ------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons polled through NVML every `period`
    seconds in a background thread; summary() keeps the samples taken inside
    [mark_start, mark_end] (the timed region)."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu_index=0, period=0.002):
        self.gpu, self.period = gpu_index, period
        self.samples = []
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self._th = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.perf_counter(), sm, rs))
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._th = threading.Thread(target=run, daemon=True)
            self._th.start()
        except Exception:
            self._th = None
        return self

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=1)

    def summary(self):
        smp = [s for s in self.samples if self.t0 is not None and self.t0 <= s[0] <= (self.t1 or 1e30)]
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted(n for n, bit in self.NAMES.items() if any(s[2] & bit for s in smp))
        return {"sm_mhz": statistics.median(s[1] for s in smp), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(smp), "source": "NVML, polled every 2 ms inside the timed region"}


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


# ------------------------------------------------------------- CPU baseline
def _ref_layer_seconds(cfg, snap, threads, groups, reps=3, warmup=1):
    """The reference's run_iteration(tree, Flatten, 128, pool, queries,
    {d_head, n_heads, tile 32, float}) over `groups` kv-head groups of one
    layer (each group: G q heads over its kv head, GQA expanded to MHA, the
    reference being MHA-only), compiled in place (oracle/_ref); else the C port
    (1 thread).  Returns (best seconds for the groups, kind, threads used)."""
    from oracle import core, ref
    G = cfg["h_q"] // cfg["h_kv"]
    d = cfg["d"]
    if ref.available():
        ref.set_threads(threads)
        ref.tune_malloc()
        inst = ref.Instance.gqa(snap, d, G * groups, groups, 42)
        for _ in range(warmup):
            inst.run_iteration(128)
        secs = [inst.run_iteration(128)[2] for _ in range(reps)]
        return min(secs), "reference", threads
    tr = core.Tree.from_snapshot(snap)
    c = core.Content.synth(tr, d * groups, 42, qdim=G * groups * d).expanded(d, G * groups, groups)
    t0 = time.perf_counter()
    core.run_iteration_flatten(tr, c, d, G * groups)
    return time.perf_counter() - t0, "port", 1


def cpu_baseline(cfg, snap, world=1):
    """CPU reference beside the GPU number (rank 0, N = 1): one layer of the
    step at all host threads (all local kv groups) and one kv group at one
    thread, each scaled to the whole step (x n_layers, x groups)."""
    nproc = os.cpu_count() or 1
    n_loc = local_kv_heads(cfg, world)
    L = cfg["n_layers"]
    t_all, kind, cores = _ref_layer_seconds(cfg, snap, nproc, n_loc, reps=3)
    t_one, _, _ = _ref_layer_seconds(cfg, snap, 1, 1, reps=1, warmup=0)
    G = cfg["h_q"] // cfg["h_kv"]
    return {"value": t_all * 1e6 * L, "unit": "us/decode step", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(), "nproc": nproc,
            "sample": f"1 layer (all {n_loc} kv-head groups x {G} q heads, GQA-expanded MHA) of run_iteration(Flatten, 128), "
                      f"best of 3 after 1 warm-up, x{L} layers (extrapolated: layers are identical work)",
            "extrapolated": {"layers": L},
            "single_thread": {"value": t_one * 1e6 * n_loc * L, "unit": "us/decode step", "cores": 1,
                              "sample": f"1 kv-head group of 1 layer at TREEATTN_THREADS=1, x{n_loc} groups x{L} layers",
                              "extrapolated": {"groups": n_loc, "layers": L}}}


# ------------------------------------------------------------------- our arm
def measure(name, cfg, args, world, rank, local_rank, clocks=None, with_cpu=False, steps=None):
    """Builds the config's tree, pools and queries on this rank, times the
    decode step (graph-replayed layer calls after ta_prepare), the per-layer
    attention time and the e2e host-buffer step.  Returns a dict."""
    import torch
    from paper_2404_00242_b200 import TreeAttention

    steps = steps or args.steps
    snap = build_snapshot(cfg)
    h_kv, h_q, d, L_layers = cfg["h_kv"], cfg["h_q"], cfg["d"], cfg["n_layers"]
    n_loc = local_kv_heads(cfg, world)
    assert cfg.get("n_local_kv_heads") or h_kv % world == 0, "kv heads must divide across ranks"
    G = h_q // h_kv
    kv_begin = (rank * n_loc) % h_kv
    root, ids, par, cnt = snap
    pages = int(sum((int(c) + 15) // 16 for c in cnt)) + 16
    ctx = TreeAttention(n_layers=L_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype=cfg["dtype"],
                        out_dtype=cfg["dtype"], max_pages=pages, device=local_rank,
                        kv_head_begin=kv_begin, n_local_kv_heads=n_loc)
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
        # a prepare of an unchanged tree is a no-op (ta_prepare keeps the
        # schedule); the headline step re-plans and re-uploads every step, as
        # after a tree change (any schedule option marks the context stale)
        ctx.set_option("tile_groups", 8)
        ctx.prepare(128, stream)
        if graph is not None:
            graph.replay()
        else:
            layers()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    io = ctx.io_stats()
    launches_per_attend = ctx.launches_per_attend()

    # ---- timed region: device time via CUDA events, max over ranks
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark_start()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark_end()
    if world > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-layer time of ta_attend on the launching stream: the graph of
    # n_layers calls, replayed back to back (each layer's KV > L2 apart)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.prepare(128, stream)
    torch.cuda.synchronize()
    reps = 10
    ev0.record(stream)
    for _ in range(reps):
        if graph is not None:
            graph.replay()
        else:
            layers()
    ev1.record(stream)
    torch.cuda.synchronize()
    attend_ms = ev0.elapsed_time(ev1) / (reps * L_layers)

    # ---- the same layer calls WITHOUT programmatic dependent launch: each
    # attention launch starts only after the previous one has completed, as
    # in a model where o_proj / MLP kernels run between the layers' attention
    # calls (no prologue / tail overlap between consecutive attention launches)
    no_overlap_ms = None
    if graph is not None:
        ctx.set_option("pdl", 0)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            layers()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(reps):
            g2.replay()
        ev1.record(stream)
        torch.cuda.synchronize()
        no_overlap_ms = ev0.elapsed_time(ev1) / (reps * L_layers)
        ctx.set_option("pdl", 1)
        del g2

    # ---- e2e through the public host-buffer entry (H2D q + D2H out per layer)
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        oh = torch.empty(out.shape, dtype=dt).pin_memory()
        qn = qh.view(torch.int16).numpy() if dt == torch.bfloat16 else qh.numpy()
        on = oh.view(torch.int16).numpy() if dt == torch.bfloat16 else oh.numpy()

        def step_host():
            # one decode step through the host-buffer entry: the n_layers
            # calls pipeline copy-in / attention / copy-out; the NEXT step's
            # ta_prepare (host plan + schedule + stream-ordered upload) runs
            # while this step's layers execute -- the next tree is known before
            # this step's outputs (one more token per leaf); the step ends when
            # every layer's output is back in host memory
            for layer in range(L_layers):
                ctx.attend_host_async(layer, qn[layer], on[layer], stream=stream)
            ctx.set_option("tile_groups", 8)   # re-plan and re-upload, as in the device-timed step
            ctx.prepare(128, stream)
            ctx.attend_host_wait()

        ctx.prepare(128, stream)
        for _ in range(2):
            step_host()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        t0 = time.perf_counter()
        for _ in range(steps):
            step_host()
        h1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1000 / steps
        ems = max(h0.elapsed_time(h1) / steps, wall_ms)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": ems * 1000.0, "unit": "us/decode step",
               "h2d_bytes_per_step": int(q.numel() * q.element_size()),
               "d2h_bytes_per_step": int(out.numel() * out.element_size()),
               "path": "ta_attend_host_async per layer (pinned host q in, host out back; copy-in, attention and "
                        "copy-out of consecutive layers overlap), the next step's ta_prepare while they run, "
                        "ta_attend_host_wait"}

    peak, peak_kind = measured_peaks()
    alg_bytes = io.kv_bytes  # one pass over unique tree KV per layer (this rank's heads)
    achieved = alg_bytes / (attend_ms * 1e-3) / 1e9
    # the bound: HBM unless the masked-in flops per unique KV byte reach the
    # ridge (the speculative configs at t >= 64 and 70B)
    tpeak, tpeak_kind = measured_tensor_peak()
    ridge = tpeak * 1e12 / (peak * 1e9)
    hbm_line = {"achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak}
    tflops = io.flops / (attend_ms * 1e-3) / 1e12
    tensor_line = {"achieved": tflops, "peak": tpeak, "peak_kind": tpeak_kind, "unit": "TFLOP/s",
                   "frac": tflops / tpeak}
    tensor_bound = io.flops >= ridge * alg_bytes
    roofline = dict(tensor_line if tensor_bound else hbm_line)
    roofline.update({"kernel": "ta_attend (attn_mma with the fused merge, or attn_fma + merge), per layer, graph-replayed",
                     "bound": "tensor" if tensor_bound else "hbm",
                     "traffic": profile_traffic(name), "alg_bytes_per_launch": alg_bytes,
                     "alg_flops_per_launch": io.flops, "intensity_flop_per_byte": io.flops / max(1, alg_bytes),
                     "other": tensor_line if not tensor_bound else hbm_line})
    if no_overlap_ms:   # the same fraction when consecutive attention launches do not overlap
        roofline["frac_no_launch_overlap"] = roofline["frac"] * attend_ms / no_overlap_ms
    res = {"value": ms * 1000.0, "ms_per_step": ms, "us_per_layer": attend_ms * 1000.0,
           "us_per_layer_no_launch_overlap": no_overlap_ms * 1000.0 if no_overlap_ms else None,
           "roofline": roofline,
           "e2e": e2e, "kv_io_bytes_per_step": io.kv_bytes * L_layers,
           "kv_bytes_loaded_per_step": io.kv_bytes_loaded * L_layers,
           "partial_io_bytes_per_step": io.partial_bytes * L_layers, "meta_bytes_per_step": io.meta_bytes,
           "q_out_bytes_per_step": (io.q_bytes + io.out_bytes) * L_layers,
           "gpu_launches": steps * L_layers * launches_per_attend,
           "schedule": {"chunks": io.n_chunks, "groups": io.n_groups, "units": io.n_units,
                        "units_mma": io.n_units_mma, "partials": io.n_partials,
                        "kv_bytes_loaded_per_layer": io.kv_bytes_loaded, "launches_per_layer": launches_per_attend},
           "config": config_obj(name, cfg, world)}
    if with_cpu and world == 1 and not args.no_cpu_baseline:
        try:
            res["cpu_baseline"] = cpu_baseline(cfg, snap, world)
        except Exception as e:  # the baseline must never sink the bench line
            res["cpu_baseline"] = {"value": None, "unit": "us/decode step", "cores": 0, "kind": "unavailable",
                                   "sample": str(e)[:200]}
    del graph, ctx
    torch.cuda.empty_cache()
    return res


def measure_decode_loop(name, cfg, args, world, rank, local_rank):
    """A real decode loop of gen_few_shot (workloads.hpp:98-111): every step
    appends one token per leaf (ta_tree_append_leaves), re-plans
    (ta_prepare: flatten plan + device schedule + metadata upload), and replays
    ONE CUDA graph of n_layers x (ta_kv_append of the step's new K/V rows +
    ta_attend).  The graph is captured once and stays valid across re-plans
    (re-captured only when ta_graph_epoch changes).  The timed steps end at the
    config's iteration (400 for B).  New K/V rows are random device tensors
    reused every step (their values do not affect the timing)."""
    import torch
    from oracle import core
    from paper_2404_00242_b200 import TreeAttention
    K, W = args.steps, max(3, args.warmup)
    it0 = cfg["iteration"] - K - W
    t = core.Tree(cfg["prefix"])
    kids = t.branch(t.root, [it0] * cfg["branches"])
    root, ids, par, cnt = t.snapshot()
    h_kv, h_q, d, L_layers = cfg["h_kv"], cfg["h_q"], cfg["d"], cfg["n_layers"]
    n_loc = local_kv_heads(cfg, world)
    G = h_q // h_kv
    pages = cfg["prefix"] // 16 + 1 + cfg["branches"] * ((cfg["iteration"] + 15) // 16 + 1) + 16
    ctx = TreeAttention(n_layers=L_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype=cfg["dtype"],
                        out_dtype=cfg["dtype"], max_pages=pages, device=local_rank,
                        kv_head_begin=(rank * n_loc) % h_kv, n_local_kv_heads=n_loc)
    for kv in args.opt:
        k_, v_ = kv.split("=")
        ctx.set_option(k_, int(v_))
    ctx.restore(root, ids, par, cnt)
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    gen = torch.Generator(device="cuda").manual_seed(99 + rank)
    for layer in range(L_layers):
        for node, c in zip(ids, cnt):
            if int(c):
                ctx.write_kv(layer, int(node), (torch.rand((int(c), n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt),
                             (torch.rand((int(c), n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt))
    L = len(ctx.leaves())
    q = (torch.rand((L_layers, L, n_loc * G, d), generator=gen, device="cuda") * 2 - 1).to(dt)
    out = torch.empty_like(q)
    nk = (torch.rand((L_layers, L, n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt)
    nv = (torch.rand((L_layers, L, n_loc, d), generator=gen, device="cuda") * 2 - 1).to(dt)
    stream = torch.cuda.current_stream()
    state = {"graph": None, "epoch": None, "recaptures": 0}

    def layers():
        s = torch.cuda.current_stream()
        for layer in range(L_layers):
            ctx.kv_append(layer, nk[layer], nv[layer], stream=s)
            ctx.attend(layer, q[layer], out[layer], stream=s)

    host = []

    prep = []

    def step():
        h0 = time.perf_counter()
        ctx.append_leaves()
        h1 = time.perf_counter()
        ctx.prepare(128, stream)
        h2 = time.perf_counter()
        host.append(h2 - h0)
        prep.append(h2 - h1)
        if state["graph"] is None or ctx.graph_epoch() != state["epoch"]:
            torch.cuda.synchronize()
            state["epoch"] = ctx.graph_epoch()
            state["graph"] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(state["graph"]):
                layers()
            state["recaptures"] += 1
        state["graph"].replay()

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    host.clear()
    prep.clear()
    fast0 = ctx.fast_prepares()
    # tcgen05 path (bf16, d 128) with the fused merge: ta_kv_append is fused into ta_attend
    fused_append = (cfg["dtype"] == "bf16" and d == 128 and
                    not any(o in args.opt for o in ("fuse_append=0", "fused_merge=0", "use_mma=0")))
    rec0 = state["recaptures"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    w0 = time.perf_counter()
    for _ in range(K):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / K
    ms = e0.elapsed_time(e1) / K
    io = ctx.io_stats()
    res = {"us_per_step": ms * 1000.0, "wall_us_per_step": wall * 1e6,
           "host_append_prepare_us_incl_backpressure": {"median": statistics.median(host) * 1e6, "max": max(host) * 1e6},
           "host_prepare_us": {"plan": io.host_plan_ns / 1e3, "schedule": io.host_schedule_ns / 1e3,
                               "upload": io.host_upload_ns / 1e3,
                               "total": (io.host_plan_ns + io.host_schedule_ns + io.host_upload_ns) / 1e3},
           "iterations": [it0 + W + 1, it0 + W + K], "graph_recaptures_in_timed_steps": state["recaptures"] - rec0,
           "kv_append_rows_per_step": ctx.kv_append_rows(),
           # ta_kv_append launches a kernel only where it is not fused into ta_attend (tcgen05 + fused merge)
           "gpu_launches_per_step": L_layers * (ctx.launches_per_attend() + (0 if fused_append else 1)),
           "fast_prepares_in_timed_steps": ctx.fast_prepares() - fast0,
           "host_prepare_us_per_step_incl_backpressure": {"median": statistics.median(prep) * 1e6, "max": max(prep) * 1e6},
           "kv_bytes_per_layer_at_end": io.kv_bytes,
           "path": "per step: ta_tree_append_leaves (1 token per leaf) + ta_prepare, then one graph replay of "
                   "n_layers x (ta_kv_append + ta_attend; the append fused into the attention launch on the tcgen05 path)"}
    del state, ctx
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------- prefix split (§8e)
def measure_prefix_split(name, cfg, args, world, rank, local_rank):
    """The optional cross-GPU split of the flattened tree (SURVEY §8e,
    paper_2404_00242_b200/prefix_split.py): every rank attends ALL kv heads
    over 1/world of the flattened tokens, then one NCCL all-to-all by head
    slice and ta_lse_merge.  Per-step device time (max over ranks) beside the
    head-sharded step of the same config."""
    import torch
    import torch.distributed as dist
    from paper_2404_00242_b200.prefix_split import PrefixSplitAttention
    snap = build_snapshot(cfg)
    root, ids, par, cnt = snap
    h_kv, h_q, d, L_layers = cfg["h_kv"], cfg["h_q"], cfg["d"], cfg["n_layers"]
    pages = int(sum((int(c) + 15) // 16 for c in cnt)) // world + len(ids) + 16
    ps = PrefixSplitAttention(snap, rank, world, n_layers=L_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d,
                              kv_dtype=cfg["dtype"], max_pages=pages, device=local_rank)
    gen = torch.Generator(device="cuda").manual_seed(7)
    for layer in range(L_layers):
        for i, n in enumerate(ids):
            off, cn = (int(x) for x in ps.ranges[i])
            if cn:   # this rank's slice of the node's KV (values do not change the work)
                ps.ctx.write_kv(layer, int(n), (torch.rand((cn, h_kv, d), generator=gen, device="cuda") * 2 - 1).bfloat16(),
                                (torch.rand((cn, h_kv, d), generator=gen, device="cuda") * 2 - 1).bfloat16())
    L = len(ps.ctx.leaves())
    q = (torch.rand((L_layers, L, h_q, d), generator=gen, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty((L_layers, L, h_q // world, d), dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        ps.ctx.prepare(128, stream)
        for layer in range(L_layers):
            ps.attend(layer, q[layer], out[layer], stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = min(args.steps, 10)
    e0.record(stream)
    for _ in range(K):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / K], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    io = ps.ctx.io_stats()
    return {"us_per_step": float(t.item()) * 1e3, "tokens_per_rank": int(sum(int(c) for _, c in ps.ranges)),
            "exchange_bytes_per_layer_per_rank": L * h_q * (d + 1) * 4 * (world - 1) // world,
            "kv_bytes_per_layer_per_rank": io.kv_bytes,
            "path": "per layer: ta_attend over this rank's token range (all heads, fp32 partials + lse), "
                    "NCCL all_to_all_single by head slice, ta_lse_merge -> this rank's heads (bf16)"}


# ------------------------------------------------ external B200 baseline
def external_baseline(timeout=600):
    """flashinfer's two-level cascade and plain paged decode on config B's tree
    (scripts/flashinfer_baseline.py), same GPU, same shapes:
    library kernels as a comparison point, run in a subprocess so a JIT or
    import failure cannot take the bench line with it."""
    import subprocess
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "flashinfer_baseline.py")],
                           capture_output=True, text=True, timeout=timeout)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-300:]}
    except Exception as e:   # noqa: BLE001 -- a baseline must never sink the line
        return {"error": str(e)[:300]}


# ---------------------------------------------------------- trace replay
# Paper Table 10 (end-to-end KV IO, TB, DeFT-Flatten; Llama-3-8B counted as 32
# heads, io_model.hpp:144-146) and Table 8 (attention latency, s, A100 80GB),
# PAPER.md:1393, 1450.
PAPER_TABLE10_TB = {"few_shot_b20": 1.68, "few_shot_b30": 2.10, "few_shot_b50": 2.94, "sorting": 12.40,
                    "document": 10.57, "keyword": 0.58, "set": 1.04, "spec_t32": 4.10, "spec_t64": 4.11,
                    "spec_t128": 4.16, "spec_t256": 4.35}
PAPER_TABLE8_S = {"few_shot_b20": 3.47, "few_shot_b30": 4.07, "few_shot_b50": 5.87, "sorting": 28.41,
                  "document": 21.45, "keyword": 2.57, "set": 3.83, "spec_t32": 13.15, "spec_t64": 16.79,
                  "spec_t128": 24.46, "spec_t256": 40.56}
REPLAY_PRESETS = ["few_shot_b20", "few_shot_b30", "few_shot_b50", "sorting", "document", "keyword", "set",
                  "spec_t32", "spec_t64", "spec_t128", "spec_t256"]


def replay_trace(preset, args, local_rank=0, n_layers=32, h_q=32, h_kv=8, d=128):
    """Trace replay: every iteration of the reference's
    preset trace (presets.hpp:29-62, generated by the compiled reference in
    oracle/_ref -- topology only, outside the timed work) is restored on the
    device context, planned (ta_prepare) and attended for all n_layers
    (Llama-3-8B shapes, bf16, GQA 32/8).  Sums the device attention time and
    the KV IO the kernels read (unique tree KV per layer, 8 kv heads), and
    beside them the reference's io_analytical(Flatten) in the paper's units
    (32 heads, io_model.hpp:88-153) against Table 10.  KV contents are not
    written (they do not change the work); the per-step events bracket only
    the n_layers attention launches."""
    import torch
    from oracle import ref
    from paper_2404_00242_b200 import TreeAttention
    snaps = ref.preset(preset)
    max_pages = max(int(sum((int(c) + 15) // 16 for c in s[3])) for s in snaps) + 16
    max_leaves = max(len(ref.leaves(s)) for s in snaps)
    ctx = TreeAttention(n_layers=n_layers, n_q_heads=h_q, n_kv_heads=h_kv, d_head=d, kv_dtype="bf16",
                        out_dtype="bf16", max_pages=max_pages, device=local_rank)
    for kv in args.opt:
        k_, v_ = kv.split("=")
        ctx.set_option(k_, int(v_))
    q = (torch.rand((n_layers, max_leaves, h_q, d), device="cuda") * 2 - 1).bfloat16()
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    evs = []
    ms_done = 0.0
    kv_dev = part_dev = 0
    kv_paper = 0
    steps = 0
    t_host = time.perf_counter()
    for snap in snaps:
        ctx.restore(*snap)
        L = len(ctx.leaves())
        if L == 0:
            continue
        ctx.prepare(128, stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for layer in range(n_layers):
            ctx.attend(layer, q[layer, :L], out[layer, :L], stream=stream)
        e1.record(stream)
        evs.append((e0, e1))
        io = ctx.io_stats()
        kv_dev += io.kv_bytes * n_layers
        part_dev += io.partial_bytes * n_layers
        kv_paper += ctx.io_analytical("flatten", 128, d, h_q, n_layers, 2)[0]
        steps += 1
        if len(evs) >= 256:   # bound the outstanding events
            torch.cuda.synchronize()
            ms_done += sum(a.elapsed_time(b) for a, b in evs)
            evs = []
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_host
    ms = ms_done + sum(a.elapsed_time(b) for a, b in evs)
    res = {"iterations": steps, "attention_s": ms / 1e3,
           "paper_table8_s_a100": PAPER_TABLE8_S.get(preset),
           "kv_io_TB_device": kv_dev / 1e12,
           "kv_io_TB_paper_units": kv_paper / 1e12,
           "paper_table10_TB": PAPER_TABLE10_TB.get(preset),
           "partial_io_TB_device": part_dev / 1e12,
           "wall_s_incl_host_restore_prepare": wall,
           "note": "kv_io_TB_device = unique tree KV read once per layer (8 kv heads, bf16): what the kernels "
                   "stream; kv_io_TB_paper_units = io_analytical(Flatten) with 32 heads (the paper's "
                   "accounting, Table 10); attention_s = sum of per-step device time of the n_layers launches"}
    del ctx
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------- main
def reference_arm(args, cfg, world):
    """The reference's own CPU path (oracle/_ref: run_iteration compiled from
    /root/reference) on this config, all host threads.  Each step times one
    layer's run_iteration over every kv-head group (the reference is MHA only:
    KV expanded to the q heads); the step value is that x n_layers, labelled
    as extrapolated (the layers are identical work)."""
    from oracle import ref
    snap = build_snapshot(cfg)
    nproc = os.cpu_count() or 1
    n_loc = local_kv_heads(cfg, world) if world == 1 else cfg["h_kv"]
    G = cfg["h_q"] // cfg["h_kv"]
    L = cfg["n_layers"]
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref was not built (needs /root/reference)"}))
        return
    ref.set_threads(nproc)
    ref.tune_malloc()
    inst = ref.Instance.gqa(snap, cfg["d"], G * n_loc, n_loc, 42)
    for _ in range(args.warmup):
        inst.run_iteration(128)
    secs = [inst.run_iteration(128)[2] for _ in range(args.steps)]
    per_layer_us = statistics.median(secs) * 1e6
    v = per_layer_us * L
    sample = (f"per step: 1 layer's run_iteration(Flatten, 128) over all {n_loc} kv-head groups "
              f"({G * n_loc} q heads, KV GQA-expanded), timed; x{L} layers")
    line = {"metric": METRIC, "value": v, "unit": "us/decode step", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v / 1000.0, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference synth.hpp content, seed 42)",
            "impl": "reference", "config": config_obj(args.config, cfg, world),
            "us_per_layer": per_layer_us, "extrapolated": {"layers": L},
            "cpu_baseline": {"value": v, "unit": "us/decode step", "cores": nproc, "kind": "reference",
                             "cpu_model": cpu_model(), "sample": sample, "extrapolated": {"layers": L}},
            "e2e": {"value": v, "unit": "us/decode step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="few_shot", choices=sorted(CONFIGS))
    ap.add_argument("--headline-only", action="store_true", help="skip the per-config sub-map")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the layer calls eagerly (no CUDA graph)")
    ap.add_argument("--opt", action="append", default=[], help="ta_set_option key=value (repeatable)")
    ap.add_argument("--replay", default=None,
                    help="comma-separated reference presets to replay end to end (or 'all'); prints one JSON line")
    ap.add_argument("--no-replay", action="store_true", help="skip the trace replays in the default run")
    ap.add_argument("--prefix-split", action="store_true",
                    help="also time the cross-GPU split of the flattened tree (all heads per rank, NCCL all-to-all "
                         "+ LSE merge) for the config; needs torchrun (N >= 1)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg, world)
        return

    import torch
    # TA_BENCH_SHARE_GPU=1 (testing the N > 1 code path on a box with fewer
    # GPUs than ranks): ranks share devices round-robin and talk over gloo
    share = os.environ.get("TA_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    if args.replay:
        names = REPLAY_PRESETS if args.replay == "all" else args.replay.split(",")
        print(json.dumps({"trace_replay": {n: replay_trace(n, args, local_rank) for n in names}}))
        return
    if world > 1 or (args.prefix_split and "RANK" in os.environ):
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    with ClockSampler(local_rank) as clocks:
        head = measure(args.config, cfg, args, world, rank, local_rank, clocks=clocks, with_cpu=True)
    decode = None
    if cfg["kind"] == "few_shot" and not args.headline_only:
        try:
            decode = measure_decode_loop(args.config, cfg, args, world, rank, local_rank)
        except Exception as e:
            decode = {"error": str(e)[:300]}
    subs = {}
    if world == 1 and not args.headline_only and args.config == "few_shot":
        for name in SUB_CONFIGS:
            try:
                subs[name] = measure(name, CONFIGS[name], args, world, rank, local_rank, with_cpu=True,
                                     steps=min(args.steps, 20))
            except Exception as e:   # a sub-config must never sink the headline line
                subs[name] = {"error": str(e)[:300]}
    split = None
    if args.prefix_split and torch.distributed.is_initialized():
        try:
            split = measure_prefix_split(args.config, cfg, args, world, rank, local_rank)
        except Exception as e:
            split = {"error": str(e)[:300]}
    external = None
    if world == 1 and not args.headline_only and args.config == "few_shot":
        external = external_baseline()
    replays = {}
    if world == 1 and not args.headline_only and not args.no_replay and args.config == "few_shot":
        for name in REPLAY_PRESETS:
            try:
                replays[name] = replay_trace(name, args, local_rank)
            except Exception as e:
                replays[name] = {"error": str(e)[:300]}
    if rank != 0:
        if torch.distributed.is_initialized():
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC,
        "value": head["value"],
        "unit": "us/decode step",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": "synthetic (uniform(-1,1) KV/Q, reference tree generators)",
        "config": head["config"],
        "kv_io_bytes_per_step": head["kv_io_bytes_per_step"],
        "partial_io_bytes_per_step": head["partial_io_bytes_per_step"],
        "meta_bytes_per_step": head["meta_bytes_per_step"],
        "us_per_layer": head["us_per_layer"],
        "us_per_layer_no_launch_overlap": head.get("us_per_layer_no_launch_overlap"),
        "roofline": head["roofline"],
        "cpu_baseline": head.get("cpu_baseline"),
        "e2e": head["e2e"],
        "clocks": clocks.summary(),
        "gpu_launches": head["gpu_launches"],
        "schedule": head["schedule"],
    }
    if decode:
        line["decode_loop"] = decode
    if subs:
        line["configs"] = subs
    if replays:
        line["trace_replay"] = replays
    if split:
        line["prefix_split"] = split
    if external:
        line["external_baseline"] = external
    print(json.dumps(line))
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def config_obj(name, cfg, world):
    n_loc = cfg.get("n_local_kv_heads") or cfg["h_kv"] // world
    par = (f"kv-head shard: {n_loc} of {cfg['h_kv']} kv heads per GPU" if cfg.get("n_local_kv_heads")
           else f"kv-head shard x{world}" if world > 1 else "single GPU")
    return {"workload": name, **{k: v for k, v in cfg.items() if k != "kind"}, "block_size": 128,
            "parallelism": par, "l2": "inputs larger than L2 (per-layer KV pools, n_layers x unique KV per step)"}


if __name__ == "__main__":
    main()
