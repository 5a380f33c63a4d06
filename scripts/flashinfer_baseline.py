"""External B200 baseline: flashinfer's two-level cascade
attention (MultiLevelCascadeAttentionWrapper, flashinfer/cascade.py) on the
few-shot tree of config B -- level 0: the 4,000-token prompt shared by all 50
queries, level 1: each query's own 400-token branch -- and flashinfer's plain
paged decode (BatchDecodeWithPagedKVCacheWrapper, every query reading its whole
path: the Flash-Decoding / Radix row of paper Table 10).  Library kernels, not
this framework's path: a comparison point on the same GPU, same shapes
(Llama-3-8B: 32 q / 8 kv heads, d 128, bf16), 32 layers with their own KV
(larger than L2), CUDA-graph-free eager timing of n_layers run() calls.

    python scripts/flashinfer_baseline.py [--layers 32] [--reps 20]
Prints one JSON line."""
import argparse
import json
import sys

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--prefix", type=int, default=4000)
    ap.add_argument("--branches", type=int, default=50)
    ap.add_argument("--branch_len", type=int, default=400)
    args = ap.parse_args()
    import flashinfer
    hq, hkv, d, P = 32, 8, 128, 16
    B, pre, br = args.branches, args.prefix, args.branch_len
    n_pre, n_br = (pre + P - 1) // P, (br + P - 1) // P
    pages = n_pre + B * n_br
    dev = "cuda"
    caches = [torch.randn(pages, 2, P, hkv, d, dtype=torch.bfloat16, device=dev) for _ in range(args.layers)]
    q = torch.randn(args.layers, B, hq, d, dtype=torch.bfloat16, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {"workload": f"few_shot {pre} + {B} x {br}, {args.layers} layers, 32/8 heads d128 bf16", "flashinfer": flashinfer.__version__}

    # --- two-level cascade (shared prefix once, then each branch)
    cas = flashinfer.MultiLevelCascadeAttentionWrapper(2, ws, "NHD")
    qo = [torch.tensor([0, B], **i32), torch.arange(B + 1, **i32)]
    kvp = [torch.tensor([0, n_pre], **i32), torch.arange(B + 1, **i32) * n_br]
    kvi = [torch.arange(n_pre, **i32), n_pre + torch.arange(B * n_br, **i32)]
    last = [torch.tensor([pre - (n_pre - 1) * P], **i32), torch.full((B,), br - (n_br - 1) * P, **i32)]
    cas.plan(qo, kvp, kvi, last, hq, hkv, d, P, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)

    def time_it(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (args.reps * args.layers)

    def run_cascade():
        for layer in range(args.layers):
            cas.run(q[layer], caches[layer])
    res["cascade_us_per_layer"] = time_it(run_cascade)

    # --- plain paged decode: every query reads prefix + its branch
    dec = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    ind = torch.cat([torch.cat([torch.arange(n_pre, **i32), n_pre + b * n_br + torch.arange(n_br, **i32)]) for b in range(B)])
    dec.plan(torch.arange(B + 1, **i32) * (n_pre + n_br), ind, torch.full((B,), br - (n_br - 1) * P, **i32), hq, hkv, d, P,
             q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)

    def run_decode():
        for layer in range(args.layers):
            dec.run(q[layer], caches[layer])
    res["paged_decode_us_per_layer"] = time_it(run_decode)
    # correctness cross-check of the two flashinfer paths on layer 0
    o1 = cas.run(q[0], caches[0]).float()
    o2 = dec.run(q[0], caches[0]).float()
    res["cascade_vs_decode_max_abs"] = float((o1 - o2).abs().max())
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
