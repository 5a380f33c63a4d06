"""Trace replay IO on the host: the reference's preset
traces (presets.hpp:29-62, from the compiled reference), summed over every
iteration with this framework's io_analytical (io_model.hpp:88-153), reproduce
the paper's Table 10 end-to-end KV IO for few-shot prompting (PAPER.md:1442,
1450: DeFT-Flatten 1.68 / 2.10 / 2.94 TB, Flash-Decoding 17.62 / 26.43 /
44.05 TB at b = 20 / 30 / 50).  The reference's reasoning and speculative
presets are its own synthetic stand-ins, so only their internal
consistency is checked: the device schedule reads exactly one pass over the
tree's KV per layer, io_analytical(Flatten) with the kv heads."""
import pytest

import bench
from oracle import ref
from paper_2404_00242_b200 import TreeAttention

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref (compiled reference) not built")

TABLE10_FLASH_DECODING = {"few_shot_b20": 17.62, "few_shot_b30": 26.43, "few_shot_b50": 44.05}


def _total(snaps, algorithm, ctx, n_heads=32):
    tot = 0
    for s in snaps:
        ctx.restore(*s)
        if len(ctx.leaves()):
            tot += ctx.io_analytical(algorithm, 128, 128, n_heads, 32, 2)[0]
    return tot / 1e12


@needs_ref
@pytest.mark.parametrize("preset", ["few_shot_b20", "few_shot_b30", "few_shot_b50"])
def test_few_shot_trace_io_matches_table10(preset):
    snaps = ref.preset(preset)
    assert len(snaps) == 400
    ctx = TreeAttention(device=-1, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype="bf16")
    assert round(_total(snaps, "flatten", ctx), 2) == bench.PAPER_TABLE10_TB[preset]
    assert round(_total(snaps, "flash-decoding", ctx), 2) == TABLE10_FLASH_DECODING[preset]


@needs_ref
@pytest.mark.parametrize("preset", ["sorting", "keyword", "spec_t64"])
def test_replay_schedule_reads_unique_kv_once(preset):
    """Every replayed iteration's device schedule covers exactly the tree's KV
    (distinct pool rows over all tiles; row blocks of a wide stripe re-read
    their stripe, from L2) and its unique KV bytes equal io_analytical(Flatten)
    with the 8 kv heads, bf16, one layer."""
    snaps = ref.preset(preset)
    ctx = TreeAttention(device=-1, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype="bf16")
    step = max(1, len(snaps) // 25)
    for s in snaps[::step]:
        ctx.restore(*s)
        if not len(ctx.leaves()):
            continue
        S = ctx.schedule(128)
        rows = set()
        for r0, info in zip(S["grp_row"], S["grp_info"]):
            rows.update(range(int(r0), int(r0) + (int(info) & 0xFF)))
        assert len(rows) * 2 * 128 * 2 * 8 == ctx.io_analytical("flatten", 128, 128, 8, 1, 2)[0]
