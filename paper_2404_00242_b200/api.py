"""Python mirror of the reference's operator API for the DeFT-Flatten path.

The reference (/root/reference/proj/include/treeattn) is a C++ header
library; its hot-path API is DecodingTree (tree.hpp) driving a PagePool
through KvLifecycle (kv_cache.hpp), partition_flatten (partition.hpp) and
run_iteration (attention.hpp:293).  ``TreeAttention`` bundles the three
behind the C ABI: the tree and its page accounting live in the native
context, the KV pages live in HBM, and attention runs on sm_100a kernels.
Method names and error behaviour follow the reference (ValueError for
std::invalid_argument, IndexError for std::out_of_range, RuntimeError for
std::logic_error).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import check, lib

_DT = {"f32": capi.TA_F32, "float32": capi.TA_F32, "bf16": capi.TA_BF16, "bfloat16": capi.TA_BF16}


def _ptr(x):
    """Device/host pointer of a torch tensor or numpy array."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        return C.c_void_p(x.ctypes.data)
    return C.c_void_p(int(x))


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


@dataclass
class IoStats:
    n_chunks: int
    n_groups: int
    n_units: int
    n_units_mma: int
    n_partials: int
    kv_bytes: int
    kv_bytes_loaded: int
    q_bytes: int
    out_bytes: int
    partial_bytes: int
    meta_bytes: int
    flops: int
    host_plan_ns: int
    host_schedule_ns: int
    host_upload_ns: int


class TreeAttention:
    """Tree KV cache + DeFT-Flatten attention on one device (one head shard).

    device=-1 gives a host-only context (tree, page accounting, planner)."""

    def __init__(self, n_layers=1, n_q_heads=1, n_kv_heads=None, d_head=64, kv_dtype="f32",
                 out_dtype="f32", page_tokens=16, max_pages=1 << 16, device=0, kv_head_begin=0,
                 n_local_kv_heads=0):
        n_kv_heads = n_q_heads if n_kv_heads is None else n_kv_heads
        s = capi.Shape(n_layers, n_q_heads, n_kv_heads, d_head, _DT[kv_dtype], _DT[out_dtype],
                       page_tokens, kv_head_begin, n_local_kv_heads, max_pages)
        h = C.c_void_p()
        check(lib().ta_ctx_create(device, C.byref(s), C.byref(h)), "ta_ctx_create")
        self._h = h
        self.n_layers, self.n_q_heads, self.n_kv_heads, self.d_head = n_layers, n_q_heads, n_kv_heads, d_head
        self.kv_dtype, self.out_dtype = kv_dtype, out_dtype
        self.page_tokens = page_tokens
        self.device = device
        self.n_local_kv_heads = n_local_kv_heads or (n_kv_heads - kv_head_begin)
        self.kv_head_begin = kv_head_begin
        self.group = n_q_heads // n_kv_heads
        self.n_local_q_heads = self.n_local_kv_heads * self.group

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib().ta_ctx_destroy(self._h)
            except Exception:   # interpreter teardown: modules already gone
                pass
            self._h = None

    def __del__(self):
        self.close()

    def set_option(self, key: str, value: int):
        check(lib().ta_set_option(self._h, key.encode(), int(value)), "ta_set_option")

    # ---------------------------------------------------------------- tree
    def new_tree(self, root_tokens: int) -> int:
        r = C.c_int32()
        check(lib().ta_tree_new(self._h, int(root_tokens), C.byref(r)), "new_tree")
        return r.value

    def restore(self, root, ids, parents, counts):
        ids = np.ascontiguousarray(ids, np.int32)
        parents = np.ascontiguousarray(parents, np.int32)
        counts = np.ascontiguousarray(counts, np.int64)
        check(lib().ta_tree_restore(self._h, int(root), len(ids), ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                    parents.ctypes.data_as(C.POINTER(C.c_int32)),
                                    counts.ctypes.data_as(C.POINTER(C.c_int64))), "restore")

    def restore_snapshot(self, snap):
        self.restore(*snap)

    def branch(self, at: int, child_token_counts) -> list[int]:
        cnt = np.ascontiguousarray(child_token_counts, np.int64)
        out = np.zeros(len(cnt), np.int32)
        check(lib().ta_tree_branch(self._h, int(at), len(cnt), cnt.ctypes.data_as(C.POINTER(C.c_int64)),
                                   out.ctypes.data_as(C.POINTER(C.c_int32))), "branch")
        return [int(x) for x in out]

    def prune(self, at: int):
        check(lib().ta_tree_prune(self._h, int(at)), "prune")

    def append_tokens(self, leaf: int, n: int):
        check(lib().ta_tree_append(self._h, int(leaf), int(n)), "append_tokens")

    def append_leaves(self, leaves=None, counts=None):
        """append_tokens on many leaves at once (default: one token on every
        leaf, leaves() order): the decode step of gen_few_shot."""
        if leaves is None:
            n = -1 if counts is None else len(counts)
            lp = None
        else:
            la = np.ascontiguousarray(leaves, np.int32)
            n, lp = len(la), la.ctypes.data_as(C.POINTER(C.c_int32))
        ca = None if counts is None else np.ascontiguousarray(counts, np.int64)
        if leaves is None and ca is not None:
            n = len(ca)
        check(lib().ta_tree_append_leaves(self._h, n, lp, None if ca is None else ca.ctypes.data_as(C.POINTER(C.c_int64))),
              "append_tokens")

    def kv_append(self, layer: int, k, v, stream=None):
        """Write this layer's KV of the tokens appended before the last
        prepare(): k, v [n_rows][n_local_kv_heads][d_head] device tensors in
        append order (one async kernel; graph-capturable)."""
        for nm, x in (("kv_append k", k), ("kv_append v", v)):
            self._check_buf(nm, x, tuple(x.shape), self.kv_dtype)
            if int(np.prod(x.shape[1:])) != self.n_local_kv_heads * self.d_head:
                raise ValueError(f"{nm}: rows must be [n_local_kv_heads][d_head]")
        check(lib().ta_kv_append(self._h, int(layer), _ptr(k), _ptr(v), _stream(stream)), "kv_append")

    def kv_append_rows(self) -> int:
        return int(lib().ta_kv_append_rows(self._h))

    def graph_epoch(self) -> int:
        """Captured ta_attend / ta_kv_append launches stay valid while this is unchanged."""
        return int(lib().ta_graph_epoch(self._h))

    def leaves(self) -> np.ndarray:
        n = C.c_int()
        check(lib().ta_tree_leaves(self._h, None, 0, C.byref(n)), "leaves")
        out = np.zeros(n.value, np.int32)
        check(lib().ta_tree_leaves(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n)),
              "leaves")
        return out

    def info(self) -> dict:
        i = capi.TreeInfo()
        check(lib().ta_tree_get_info(self._h, C.byref(i)), "info")
        return {f: getattr(i, f) for f, _ in capi.TreeInfo._fields_}

    def snapshot(self):
        n = C.c_int()
        check(lib().ta_tree_snapshot(self._h, None, None, None, 0, C.byref(n)), "snapshot")
        ids = np.zeros(n.value, np.int32)
        par = np.zeros(n.value, np.int32)
        cnt = np.zeros(n.value, np.int64)
        check(lib().ta_tree_snapshot(self._h, ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                     par.ctypes.data_as(C.POINTER(C.c_int32)),
                                     cnt.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)), "snapshot")
        return self.info()["root"], ids, par, cnt

    # ---------------------------------------------------------------- pool
    def pool_stats(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ta_pool_stats(self._h, C.byref(a), C.byref(b), C.byref(c)), "pool_stats")
        return {"page_count": a.value, "free_page_count": b.value, "live_slots": c.value}

    def token_ref(self, node: int, token: int):
        p, s = C.c_int32(), C.c_int32()
        check(lib().ta_pool_token_ref(self._h, int(node), int(token), C.byref(p), C.byref(s)), "token_ref")
        return p.value, s.value

    # ------------------------------------------------------------ checking
    def _torch_dtype(self, name):
        import torch
        return torch.bfloat16 if name in ("bf16", "bfloat16") else torch.float32

    def _check_buf(self, what, x, shape, dtype_name, device_only=True):
        """Layout contract of the C ABI: dense row-major, the context's dtype,
        the context's device.  A mismatch is the reference's invalid_argument."""
        if x is None:
            return
        if hasattr(x, "is_contiguous"):   # torch
            want = self._torch_dtype(dtype_name)
            if x.dtype != want:
                raise ValueError(f"{what}: dtype {x.dtype}, expected {want}")
            if not x.is_contiguous():
                raise ValueError(f"{what}: tensor must be contiguous")
            if device_only and (not x.is_cuda or x.device.index != self.device):
                raise ValueError(f"{what}: must be a tensor on cuda:{self.device}, got {x.device}")
            if not device_only and x.is_cuda and x.device.index != self.device:
                raise ValueError(f"{what}: on {x.device}, context is on cuda:{self.device}")
        elif isinstance(x, np.ndarray):
            if device_only:
                raise ValueError(f"{what}: expected a device tensor, got a numpy array")
            if not x.flags["C_CONTIGUOUS"]:
                raise ValueError(f"{what}: array must be C-contiguous")
            isz = 2 if dtype_name in ("bf16", "bfloat16") else 4
            if x.dtype.itemsize != isz:
                raise ValueError(f"{what}: element size {x.dtype.itemsize}, expected {isz} ({dtype_name})")
        else:
            return   # raw pointer: the caller vouches for the layout
        if tuple(x.shape) != tuple(shape) and int(np.prod(x.shape)) != int(np.prod(shape)):
            raise ValueError(f"{what}: shape {tuple(x.shape)}, expected {tuple(shape)}")

    def write_kv(self, layer: int, node: int, k, v, tok_begin: int = 0, stream=None):
        """k, v: [n_tok][n_local_kv_heads][d_head] (torch device tensor or host numpy/torch)."""
        n = int(k.shape[0])
        on_dev = bool(getattr(k, "is_cuda", False))
        for nm, x in (("write_kv k", k), ("write_kv v", v)):
            self._check_buf(nm, x, (n, self.n_local_kv_heads, self.d_head), self.kv_dtype, device_only=False)
        if bool(getattr(v, "is_cuda", False)) != on_dev:
            raise ValueError("write_kv: k and v must both be on the device or both on the host")
        check(lib().ta_kv_write(self._h, int(layer), int(node), int(tok_begin), n, _ptr(k), _ptr(v),
                                int(on_dev), _stream(stream)), "write_kv")

    # ---------------------------------------------------------------- plan
    def plan_flatten(self, block_size: int = 128) -> dict:
        """partition_flatten (partition.hpp:212-253) in oracle.core's plan format."""
        pv = capi.PlanView()
        check(lib().ta_plan_flatten(self._h, int(block_size), C.byref(pv)), "plan_flatten")
        groups = []
        for g in range(pv.n_groups):
            s0, s1 = pv.seg_begin[g], pv.seg_begin[g + 1]
            q0, q1 = pv.q_begin[g], pv.q_begin[g + 1]
            groups.append({
                "id": g,
                "segments": [(pv.seg_node[s], pv.seg_offset[s], pv.seg_len[s]) for s in range(s0, s1)],
                "queries": [pv.queries[q] for q in range(q0, q1)],
                "masks": [pv.seg_mask[s] for s in range(s0, s1)],
            })
        return {"strategy": "flatten", "block_size": pv.block_size, "groups": groups}

    def plan_json(self, block_size: int = 128) -> str:
        n = C.c_size_t()
        check(lib().ta_plan_json(self._h, int(block_size), None, 0, C.byref(n)), "plan_json")
        buf = C.create_string_buffer(n.value + 1)
        check(lib().ta_plan_json(self._h, int(block_size), buf, n.value + 1, C.byref(n)), "plan_json")
        return buf.value.decode()

    def set_strategy(self, name: str):
        """Partition strategy planned by prepare / plan_json / plan_flatten:
        "flatten" (default, the hot path), "node", "node-chunk", "q-guided"
        (partition.hpp:16; the paper's ablations on the same kernels)."""
        if name not in capi.TA_STRATEGY:
            raise ValueError("unknown strategy: " + name)
        self.set_option("strategy", capi.TA_STRATEGY[name])

    def io_measured(self, block_size, d_head, n_heads, n_layers, dtype_bytes):
        """io_measured(make_plan(tree, strategy, bs), CostParams) (io_model.hpp:158-170):
        (kv, q, mask, partial) bytes."""
        p = capi.CostParams(d_head, n_heads, n_layers, dtype_bytes)
        r = capi.IoReport()
        check(lib().ta_io_measured(self._h, int(block_size), C.byref(p), C.byref(r)), "io_measured")
        return (r.kv_bytes, r.q_bytes, r.mask_bytes, r.partial_bytes)

    def io_analytical(self, algorithm, block_size, d_head, n_heads, n_layers, dtype_bytes):
        """io_analytical(tree, algorithm, CostParams, bs) (io_model.hpp:88-153)."""
        if algorithm not in capi.TA_ALG:
            raise ValueError("unknown algorithm: " + algorithm)
        p = capi.CostParams(d_head, n_heads, n_layers, dtype_bytes)
        r = capi.IoReport()
        check(lib().ta_io_analytical(self._h, capi.TA_ALG[algorithm], C.byref(p), int(block_size), C.byref(r)),
              "io_analytical")
        return (r.kv_bytes, r.q_bytes, r.mask_bytes, r.partial_bytes)

    # ----------------------------------------------------------- attention
    def prepare(self, block_size: int = 128, stream=None):
        check(lib().ta_prepare(self._h, int(block_size), _stream(stream)), "prepare")

    def attend(self, layer: int, q, out=None, lse=None, stream=None):
        """q [L][n_local_q_heads][d_head] device tensor -> out (same layout)."""
        L = int(q.shape[0]) if hasattr(q, "shape") else None
        if L is not None:
            n = C.c_int()
            check(lib().ta_tree_leaves(self._h, None, 0, C.byref(n)), "leaves")
            if L != n.value:
                raise ValueError(f"attend q: {L} query rows, the tree has {n.value} leaves")
            shape = (L, self.n_local_q_heads, self.d_head)
            self._check_buf("attend q", q, shape, self.kv_dtype)
        if out is None:
            import torch
            out = torch.empty(shape, dtype=self._torch_dtype(self.out_dtype), device=q.device)
        elif L is not None:
            self._check_buf("attend out", out, shape, self.out_dtype)
        if lse is not None and L is not None:
            self._check_buf("attend lse", lse, (L, self.n_local_q_heads), "f32")
        check(lib().ta_attend(self._h, int(layer), _ptr(q), _ptr(out), _ptr(lse), _stream(stream)), "attend")
        return out

    def attend_host(self, layer: int, q_host, out_host, stream=None):
        check(lib().ta_attend_host(self._h, int(layer), _ptr(q_host), _ptr(out_host), _stream(stream)),
              "attend_host")
        return out_host

    def attend_host_async(self, layer: int, q_host, out_host, stream=None):
        """Pipelined host-buffer attend: returns once queued; out_host is complete
        after attend_host_wait().  Use pinned host buffers for overlap."""
        check(lib().ta_attend_host_async(self._h, int(layer), _ptr(q_host), _ptr(out_host), _stream(stream)),
              "attend_host_async")
        return out_host

    def attend_host_wait(self):
        check(lib().ta_attend_host_wait(self._h), "attend_host_wait")

    def fast_prepares(self) -> int:
        """prepare() calls that patched the schedule in place (decode-step fast path)."""
        return int(lib().ta_fast_prepares(self._h))

    def io_stats(self) -> IoStats:
        s = capi.IoStats()
        check(lib().ta_io_stats_get(self._h, C.byref(s)), "io_stats")
        return IoStats(**{f: getattr(s, f) for f, _ in capi.IoStats._fields_})

    def schedule(self, block_size: int = 128) -> dict:
        """The device schedule (see include/treeattn_b200.h, ta_schedule_view)
        as numpy arrays: items [n][8], tiles [n][4] (+ decoded ng / boxes),
        groups, slot maps, partial/merge lists, empty leaf-heads."""
        v = capi.ScheduleView()
        check(lib().ta_schedule_get(self._h, int(block_size), C.byref(v)), "schedule")

        def arr(p, n, dt=np.int64):
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt) if n else np.zeros(0, dt)
        tiles = arr(v.tiles, 4 * v.n_tiles).reshape(-1, 4)
        raw = tiles.astype(np.int32).view(np.uint8).reshape(-1, 16) if v.n_tiles else np.zeros((0, 16), np.uint8)
        n_mp = v.merge_begin[v.n_merge] if v.n_merge else 0
        return {"n_ctas": v.n_ctas, "cta_begin": arr(v.cta_begin, v.n_ctas + 1),
                "items": arr(v.items, 8 * v.n_items).reshape(-1, 8),
                "tile_grp_begin": tiles[:, 0] if v.n_tiles else np.zeros(0, np.int64),
                "tile_ng": raw[:, 4].astype(np.int64), "tile_nbox": raw[:, 5].astype(np.int64),
                "tile_boxes": raw[:, 8:16].astype(np.int64),
                "grp_row": arr(v.grp_row, v.n_grp), "grp_info": arr(v.grp_info, v.n_grp),
                "slot_leaf": arr(v.slot_leaf, v.n_slot_leaf), "slot_out": arr(v.slot_out, v.n_slot_out),
                "n_partials": v.n_partials, "part_merge": arr(v.part_merge, v.n_partials),
                "merge_leaf": arr(v.merge_leaf, v.n_merge), "merge_head": arr(v.merge_head, v.n_merge),
                "merge_begin": arr(v.merge_begin, v.n_merge + 1), "merge_parts": arr(v.merge_parts, n_mp),
                "empty": arr(v.empty, 2 * v.n_empty).reshape(-1, 2), "n_lanes": v.n_lanes,
                "use_mma": bool(v.use_mma), "fused_merge": bool(v.fused_merge),
                **self._fused_lists(v, arr)}

    @staticmethod
    def _fused_lists(v, arr):
        if not v.fused_merge:
            return {}
        pb = arr(v.cta_pub_begin, v.n_ctas + 1)
        ob = arr(v.cta_own_begin, v.n_ctas + 1)
        return {"cta_pub_begin": pb, "cta_pub": arr(v.cta_pub, 2 * int(pb[-1])).reshape(-1, 2),
                "cta_own_begin": ob, "cta_own": arr(v.cta_own, int(ob[-1]))}

    def launches_per_attend(self) -> int:
        return lib().ta_launches_per_attend(self._h)


def run_iteration(ctx: TreeAttention, layer: int, q, block_size: int = 128, lse=None, stream=None):
    """run_iteration(tree, Strategy::Flatten, block_size, pool, queries, params)
    (attention.hpp:293-334): plan + attention for one layer.  Returns
    (out [L][h][d] device tensor, plan dict)."""
    ctx.prepare(block_size, stream)
    out = ctx.attend(layer, q, lse=lse, stream=stream)
    return out, ctx.plan_flatten(block_size)
