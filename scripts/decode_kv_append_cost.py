"""Cost of the per-layer ta_kv_append launches inside the decode loop:
the bench's decode loop (config B, iterations 376-400) with and without the
kv_append calls in the replayed graph (without them the new rows' KV is
stale: timing only)."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

args = types.SimpleNamespace(steps=20, warmup=5, opt=[])
cfg = bench.CONFIGS["few_shot"]
from paper_2404_00242_b200 import api

full = bench.measure_decode_loop("few_shot", cfg, args, 1, 0, 0)
orig = api.TreeAttention.kv_append
api.TreeAttention.kv_append = lambda self, *a, **k: None
try:
    bare = bench.measure_decode_loop("few_shot", cfg, args, 1, 0, 0)
finally:
    api.TreeAttention.kv_append = orig
print(f"decode step with kv_append {full['us_per_step']:.1f} us, without {bare['us_per_step']:.1f} us, "
      f"kv_append share {full['us_per_step'] - bare['us_per_step']:.1f} us per step (32 launches)")
